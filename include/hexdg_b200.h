/*
 * hexdg_b200 -- C ABI of the B200-native FP64 DGSEM right-hand side and
 * low-storage Runge-Kutta stage update.
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (`hexdg`, pure Python + numba) has no FFI: its boundary is the Python API
 * `Domain` kernel wrappers / `RankWorker.evaluate_rhs` / `rk_step`
 * (reference pkg/src/hexdg/operator.py:494-727, parallel.py:539-563,
 * timedisc.py:114-138). Each entry point below names the reference call it
 * replaces. The Python package `paper_2404_12703_b200` binds these through
 * ctypes (paper_2404_12703_b200/_lib.py); INTEGRATION.md shows the binding a
 * maintainer of the reference would add.
 *
 * Conventions
 *  - All array pointers inside hdg_domain and all U/Ut/dU arguments are CUDA
 *    DEVICE pointers (float64 / int32), C-contiguous, in the reference's
 *    layouts: U[e][k][j][i][5], Ja[e][a][k][j][i][c], faces [s][q][p][var].
 *    The only additional device layouts are Fvis[e][a][v=1..4][k][j][i] and
 *    fvface[s][role][q][p][4].
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *    and asynchronous, performs no allocation and no host synchronisation.
 *  - Return codes: 0 ok; < 0 argument / CUDA error (message via
 *    hdg_last_error()). Admissibility failures are reported through the
 *    device status words (HDG_STATUS_*), read by the caller when it syncs, so
 *    the Python layer can raise the reference's AdmissibilityError /
 *    NumericalFailure.
 *  - `exact` != 0 selects the kernel set compiled with -fmad=false: results
 *    are bit-identical to the reference's numba kernels (except the shock
 *    indicator's exp() and the MMS source's sin/cos, within 1 ulp). exact == 0
 *    selects the FMA-contracted kernels (<= 1e-12 normwise vs the reference).
 */
#ifndef HEXDG_B200_H
#define HEXDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HDG_ABI_VERSION 2

/* orientation / side meta encoding (side_info[s*4 + 2]) */
#define HDG_SIDE_INNER 0        /* both elements local                     */
#define HDG_SIDE_BC 1           /* Dirichlet boundary side                 */
#define HDG_SIDE_MPI_PRIMARY 2  /* local primary, replica on another rank  */
#define HDG_SIDE_MPI_REPLICA 3  /* local replica, primary on another rank  */

/* status words (int32[8], device) */
#define HDG_STATUS_BAD_PRIM 0   /* cons_to_prim: rho <= 0 or p <= 0 seen   */
#define HDG_STATUS_BAD_SIDE 1   /* max local side with inadmissible trace (-1 none) */
#define HDG_STATUS_NONFINITE 2  /* non-finite U seen by hdg_local_dt       */
#define HDG_STATUS_PEER_TIMEOUT 3 /* a peer-memory exchange flag never arrived (~10 s) */

typedef struct hdg_domain {
  int32_t N;           /* polynomial degree, 1..7                          */
  int32_t node_type;   /* 0 = LGL, 1 = GL                                  */
  int32_t ne;          /* local elements                                   */
  int32_t ns;          /* local sides (reference Domain.ns)                */
  /* geometry and tables -- reference Domain attributes (operator.py:502-625) */
  const double* basis;      /* pack_basis(): D|Dhat|Dsplit|Vinv (n1*n1), w|l-|l+|lhat-|lhat+|1/w (n1) */
  const double* Ja;         /* (ne,3,n1,n1,n1,3)                            */
  const double* J;          /* (ne,n1,n1,n1)                                */
  const double* invJ;       /* (ne,n1,n1,n1) = 1.0/J                        */
  const double* nvec;       /* (ns,n1,n1,3)                                 */
  const double* ssurf;      /* (ns,n1,n1)                                   */
  const double* x;          /* (ne,n1,n1,n1,3), only for the MMS source     */
  const int32_t* ef_info;   /* (ne,6): side<<3 | is_replica<<2 | orient     */
  const int32_t* side_info; /* (ns,4): elem_p, elem_r (local or -1), meta, halo slot
                               meta = loc_p | loc_r<<3 | orient<<6 | bc<<8 | kind<<12 */
  const double* bc_states;  /* (8,5)                                        */
  const double* fvm0;       /* FV subcell interface metrics (ne,n1,n1,n1+1,3) or NULL */
  const double* fvm1;
  const double* fvm2;
  /* workspaces (device, caller-allocated) */
  double* UL;               /* (ns,n1,n1,5) traces (GL path, halo traces)   */
  double* UR;
  double* fstar;            /* (ns,n1,n1,5)                                 */
  double* Fvis;             /* (ne,3,4,n1^3)            [viscous]           */
  double* fvface;           /* (ns,2,n1,n1,4) face viscous fluxes [viscous] */
  double* g;                /* (ne,n1,n1,n1,3,4) lifted gradients, optional (API mirror) */
  double* gL;               /* (ns,n1,n1,3,4) optional (API mirror)          */
  double* gR;
  double* vstar;            /* (ns,n1,n1,4) optional (API mirror)            */
  double* alpha;            /* (ne) blending factors [shock]                */
  int32_t* status;          /* int32[8]                                     */
  uint64_t* dt_bits;        /* uint64[2]: [0] min dt as positive-double bits */
  double* vol;              /* (ne,n1,n1,n1,5) volume integral [viscous LGL path] */
  double* rfv;              /* (ne,n1,n1,n1,5) FV subcell residual of flagged elements [shock] */
  int32_t* fv_list;         /* (ne) flagged elements of the current stage (any order) [shock] */
  int32_t* fv_count;        /* int32[1] number of flagged elements [shock] */
  int32_t* work;            /* int32[4] work counters of the persistent FV kernel (reset per launch, stream-ordered) */
} hdg_domain;

typedef struct hdg_params {
  double gamma, R, Pr, mu_ref, T_ref;
  int32_t law;              /* 0 constant, 1 Sutherland                     */
  int32_t viscous;          /* mu_ref > 0                                   */
  int32_t split;            /* 1 split-form volume integral, 0 standard     */
  int32_t surf_solver;      /* 0 LLF, 1 HLLC, 2 LLF_SPLIT (DG surface flux) */
  int32_t fv_solver;        /* FV subcell interior solver (0 LLF, 1 HLLC)   */
  int32_t shock;            /* FV subcell blending on                       */
  int32_t indicator;        /* 0 Hennemann modal, 1 constant                */
  double alpha_max, alpha_min, alpha_const;
  double ind_threshold;     /* modal_threshold(N)                           */
  double ind_slope;         /* -SHARPNESS / threshold                       */
  int32_t source;           /* 1: add the MMS source (testcases.k_mms_source) */
  double mms_A, mms_a;      /* amplitude, speed                             */
  int32_t exact;            /* 1: -fmad=false kernel set                    */
  int32_t pad;
  double cfl, cfl_visc;     /* RunConfig cfl / cflvisc: the next-step dt folded into the
                               last stage (HDG_STAGE_NEXT_DT)                   */
} hdg_params;

/* ---- library ---------------------------------------------------------- */
int hdg_abi_version(void);
const char* hdg_last_error(void);
/* sizeof the two descriptor structs, for binding-side layout checks */
int64_t hdg_sizeof_domain(void);
int64_t hdg_sizeof_params(void);
/* number of kernels this library has launched so far (process-wide counter) */
int64_t hdg_launch_count(void);
/* Validates a domain descriptor (degree supported, required pointers set). */
int hdg_check_domain(const hdg_domain* d, const hdg_params* p);

/* ---- the time derivative ---------------------------------------------- */
/* RankWorker.evaluate_rhs(t) (parallel.py:539-563) for one rank with no
 * partition-boundary sides: Ut = -(1/J)(VolInt + SurfInt) [+ FV blend] [+ source].
 * `sides` lists the local sides whose flux this rank computes (Domain.sides_inner,
 * plus sides_mpi_primary once their halo traces arrived); NULL with nsides == ns
 * means every local side in order (no list indirection). LGL only; the GL path
 * is prolong + hdg_fill_flux_traces + hdg_phase_volume.
 * Ut is overwritten (the reference zeroes then accumulates). */
int hdg_rhs(const hdg_domain* d, const hdg_params* p, const double* U, double* Ut,
            double t, const int32_t* sides, int32_t nsides, void* stream);

/* `first` of hdg_stage is a bit set: bit 0 = first stage of the step; bit 1
 * (HDG_STAGE_NEXT_DT) = also evaluate k_local_dt + isfinite (src/operator.py:460-487,
 * src/parallel.py:595-604) on the UPDATED U -- the next step's _compute_dt, folded
 * into the last stage's epilogue -- min-reduced into d->dt_bits[0] (which
 * hdg_dt_finalize resets to +inf after reading) with p->cfl / p->cfl_visc. */
#define HDG_STAGE_NEXT_DT 2
/* One fused LSERK stage: RHS as hdg_rhs, then (timedisc.py:132-137)
 *   dU = first ? dt*Ut : A*dU + dt*Ut;   U += B*dU
 * with dt = time_dev[1] and stage time time_dev[0] + c*dt read on the device,
 * so a whole step can be captured in a CUDA graph. Ut is never stored. */
int hdg_stage(const hdg_domain* d, const hdg_params* p, double* U, double* dU,
              const double* time_dev, double A, double B, double c, int first,
              const int32_t* sides, int32_t nsides, void* stream);

/* Split phases of the same stage for multi-rank overlap:
 *   hdg_phase_lift   -- BR1 lifting (viscous only): Fvis + face viscous fluxes
 *                       for every local element (needs all face traces).
 *   hdg_phase_flux   -- surface fluxes f* on the given local side list.
 *   hdg_phase_volume -- volume + surface integral + Jacobian [+FV][+source]
 *                       then either store Ut (dU == NULL) or the LSERK update. */
int hdg_phase_lift(const hdg_domain* d, const hdg_params* p, const double* U, void* stream);
/* Navier-Stokes LGL path (A -> flux -> C):
 *   hdg_phase_elem   -- A: lifting + face viscous fluxes + the complete volume
 *                       integral into d->vol (k_lift_* + k_vol_int_*)
 *   hdg_phase_update -- C: Ut = -(1/J)(vol + SurfInt) [+FV blend][+source], then
 *                       store Ut or the LSERK update (same modes as phase_volume) */
int hdg_phase_elem(const hdg_domain* d, const hdg_params* p, const double* U, void* stream);
int hdg_phase_update(const hdg_domain* d, const hdg_params* p, double* U, double* Ut_or_dU,
                     const double* time_dev, double t_host, double A, double B, double c,
                     int mode, void* stream);
/* the same two phases restricted to a list of local elements (N >= 4), so a
 * partitioned run can compute interior elements while face data is in flight.
 * reset_fv: clear the flagged-element count first (first pass of a stage);
 * do_fv: run the FV residual of the flagged elements first (first pass). */
int hdg_phase_elem_list(const hdg_domain* d, const hdg_params* p, const double* U,
                        const int32_t* elems, int32_t n, int reset_fv, void* stream);
int hdg_phase_update_list(const hdg_domain* d, const hdg_params* p, double* U,
                          double* Ut_or_dU, const double* time_dev, double t_host, double A,
                          double B, double c, int mode, const int32_t* elems, int32_t n,
                          int do_fv, void* stream);
int hdg_phase_flux(const hdg_domain* d, const hdg_params* p, const double* U,
                   const int32_t* sides, int32_t nsides, int32_t solver, void* stream);
int hdg_phase_volume(const hdg_domain* d, const hdg_params* p, double* U, double* Ut_or_dU,
                     const double* time_dev, double t_host, double A, double B, double c,
                     int mode, void* stream);
#define HDG_MODE_STORE_UT 0
#define HDG_MODE_LSERK 1
#define HDG_MODE_LSERK_FIRST 2
/* mode may carry stage flags in bits 4..: (flags << 4); flags == 0 means the full
 * RHS. 1 surface integral, 2 Jacobian, 4 accumulate into Ut (Domain.vol_int),
 * 8 FV residual only (shock.fv_subcell_operator), 16 FV blend + source,
 * 32 indicator only (shock.indicator_alpha), 64 (hdg_phase_update*, LSERK modes):
 * the next step's local dt + isfinite on the updated U, as HDG_STAGE_NEXT_DT. */

/* ---- reference Domain kernel wrappers (operator.py:629-727) ------------ */
/* k_cons_to_prim: prim (ne*n1^3, 7); sets HDG_STATUS_BAD_PRIM. */
int hdg_cons_to_prim(const hdg_domain* d, const hdg_params* p, const double* U, double* prim,
                     void* stream);
/* k_prolong on rows (n,5) int32 (side, elem, loc, is_primary, orient) -> d->UL / d->UR */
int hdg_prolong(const hdg_domain* d, const double* U, const int32_t* rows, int32_t nrows,
                void* stream);
/* apply_bc_traces: UR[s] = bc_states[side_bc[s]] on the listed BC sides */
int hdg_apply_bc_traces(const hdg_domain* d, const int32_t* sides, int32_t nsides, void* stream);
/* k_fill_flux_convective (+ k_fill_flux_viscous from d->fvface) from d->UL/d->UR */
int hdg_fill_flux_traces(const hdg_domain* d, const hdg_params* p, const int32_t* sides,
                         int32_t nsides, int32_t solver, void* stream);
/* k_surf_int (gather SurfInt, operator.py:333-358): Ut += ... (raw kernel API) */
int hdg_surf_int(const hdg_domain* d, const double* fstar, double* Ut, void* stream);
/* k_apply_jac: Ut *= -1/J */
int hdg_apply_jac(const hdg_domain* d, double* Ut, void* stream);
/* k_local_dt + isfinite(U): atomically mins dt into d->dt_bits[0] and sets
 * HDG_STATUS_NONFINITE; caller zero-initialises (dt_bits[0] = +inf bits). */
int hdg_local_dt(const hdg_domain* d, const hdg_params* p, const double* U, double cfl,
                 double cfl_visc, void* stream);
/* dt finalisation on device: time_dev = [t, dt]; dt = min over ranks (already
 * reduced into dt_bits[0]); clipped to tend - t (parallel.py:649-650); then
 * dt_bits[0] = +inf, ready for the next step's (folded) local dt. */
int hdg_dt_finalize(const hdg_domain* d, double* time_dev, double tend, void* stream);
/* t += dt (parallel.py:656) on device */
int hdg_time_advance(double* time_dev, void* stream);
/* TGV analysis partial sums per element -- replaces k_analysis_partials
 * (src/testcases.py:190-226, called by testcases.analysis_partials :229-238 and
 * RankWorker.analyze src/parallel.py:606-629). out (ne, 9), row order: mass,
 * mom_x, mom_y, mom_z, energy, rho u.u, mu/mu0 |curl u|^2, mu/mu0 (div u)^2,
 * volume. g = lifted gradients (ne, n1^3, 3, 4), required when viscous. mu0 > 0
 * (the reference passes 1.0 when the case has no reference viscosity). */
int hdg_analysis_partials(const hdg_domain* d, const hdg_params* p, const double* U,
                          const double* g, double mu0, double* out, void* stream);

/* ---- generic device helpers -------------------------------------------- */
/* rk_step's numpy update (timedisc.py:132-137) as one fused pass over n doubles */
int hdg_lserk_update(double* U, double* dU, const double* Ut, int64_t n, double A, double B,
                     double dt, int first, void* stream);
/* face-block gather/scatter for the a-priori ordered exchange (parallel.py:348-377):
 * pack:   buf[k*width + w] = src[idx[k]*width + w]
 * unpack: dst[idx[k]*width + w] = buf[k*width + w] */
int hdg_pack(const double* src, const int32_t* idx, int32_t n, int32_t width, double* buf,
             void* stream);
int hdg_unpack(const double* buf, const int32_t* idx, int32_t n, int32_t width, double* dst,
               void* stream);
/* the rank's own traces of the listed partition-boundary sides, in list order
 * (send_traces payload, parallel.py:405-410): buf[k][q][p][5]; LGL gathers the
 * boundary nodes of U, GL copies the prolonged UL/UR rows */
int hdg_pack_traces(const hdg_domain* d, const double* U, const int32_t* sides, int32_t n,
                    double* buf, void* stream);

/* ---- partition-boundary exchange over NVLink peer memory ----------------- */
/* Same payloads and a-priori order as the send/recv tasks of _build_rhs
 * (parallel.py:404-499) / hdg_pack + hdg_unpack, without staging: row k of the
 * send list is written straight into row dst[k] of the destination array of
 * neighbour slot nbr[k] (dst_base[slot] = a CUDA-IPC mapped device pointer of
 * that rank's UL/UR block, fvface or fstar). The block that completes the grid
 * advances the device epoch counter *epoch of the phase and publishes it to every
 * neighbour's flag word (flag_ptrs[slot], release at system scope) after all
 * blocks fenced their stores (device counters: the calls are graph-replayable). `counter` is a private
 * uint32 advanced by gridDim.x per call (never reset; keep the row count of a
 * given counter fixed). traces: the own trace of local side src[k] (LGL, U).
 * rows: `width` doubles of row src[k] of src_rows. */
int hdg_peer_send_traces(const hdg_domain* d, const double* U, const int32_t* nbr,
                         const int32_t* src, const int32_t* dst, int32_t n, const uint64_t* dst_base,
                         const uint64_t* flag_ptrs, int32_t n_nbr, uint32_t* counter,
                         uint64_t* epoch, void* stream);
int hdg_peer_send_rows(const double* src_rows, int32_t width, const int32_t* nbr,
                       const int32_t* src, const int32_t* dst, int32_t n, const uint64_t* dst_base,
                       const uint64_t* flag_ptrs, int32_t n_nbr, uint32_t* counter,
                       uint64_t* epoch, void* stream);
/* Exchange wait fused into the consumer kernel: list positions >= pos need the
 * neighbours' payload of a phase; the kernel's blocks that reach them first
 * wait (one thread, acquire at system scope, bounded as hdg_peer_wait) until
 * flags[idx[i]] >= *epoch -- the value this rank's own send of the phase just
 * wrote to its send counter. Interior work before pos overlaps the exchange. */
typedef struct hdg_gate {
  const uint64_t* flags;
  const int32_t* idx;
  int32_t n;                /* 0 = no gate */
  int32_t pos;
  const uint64_t* epoch;
} hdg_gate;
int hdg_phase_elem_gated(const hdg_domain* d, const hdg_params* p, const double* U,
                         const int32_t* elems, int32_t n, int reset_fv, const hdg_gate* gate,
                         void* stream);
int hdg_phase_flux_gated(const hdg_domain* d, const hdg_params* p, const double* U,
                         const int32_t* sides, int32_t nsides, int32_t solver, const hdg_gate* gate,
                         void* stream);
int hdg_phase_update_gated(const hdg_domain* d, const hdg_params* p, double* U, double* out,
                           const double* time_dev, double t_host, double A, double B, double c,
                           int mode, const int32_t* elems, int32_t n, int do_fv,
                           const hdg_gate* gate, void* stream);
/* CUDA IPC of the exchange's landing arrays: export = 64-byte cudaIpcMemHandle_t
 * of the allocation containing ptr + the byte offset of ptr in it; open maps a
 * neighbour's allocation into the CURRENT device's context (peer access enabled
 * lazily) and returns its base; close unmaps. */
int hdg_ipc_export(const void* ptr, void* handle, int64_t* offset);
int hdg_ipc_open(const void* handle, void** ptr);
int hdg_ipc_close(void* ptr);
/* Stream-ordered wait until flags[idx[i]] >= *epoch for all i, *epoch = this
 * rank's send counter of the phase (its own send of the phase precedes the wait;
 * acquire, system scope; bounded: after ~10 s sets status[HDG_STATUS_PEER_TIMEOUT]). */
int hdg_peer_wait(const uint64_t* flags, const int32_t* idx, int32_t n, const uint64_t* epoch,
                  int32_t* status, void* stream);
/* _allreduce of _compute_dt (parallel.py:567-579, :595-604) over peer memory:
 * d->dt_bits[0] = min over ranks, d->status[i] = max over ranks. slot_ptrs[q] /
 * flag_ptrs[q] = rank q's (IPC-mapped) int64[2][world][10] slot array and
 * uint64[world] flag array (own rank included); my_slots / my_flags = this
 * rank's. One block; world <= 32. */
int hdg_peer_allreduce_dt(const hdg_domain* d, const uint64_t* slot_ptrs, const uint64_t* flag_ptrs,
                          const int64_t* my_slots, const uint64_t* my_flags, int32_t me,
                          int32_t world, uint64_t* epoch, void* stream);

/* ---- API-granularity calls of the reference's Python surface ------------- */
/* Point physics of hexdg.equations for n independent inputs (device arrays, row
 * per item): op 0 pt_euler_flux_dir (src/equations.py:93-102), in (rho,u,v,w,p,
 * rhoE,nx,ny,nz); op 1 pt_viscous_flux_dir (:262-285) with mu = pt_viscosity(T),
 * lam = pt_conductivity(mu), in (u,v,w,T, g[3][4], nx,ny,nz); op 2 pt_riemann
 * (:219-232) with `solver`, in (rhoL,uL,vL,wL,pL,rhoEL, rhoR,...,rhoER, nx,ny,nz);
 * op 3 pt_split_flux_kep (:235-259), in (rhoL,uL,vL,wL,pL,hL, rhoR,...,hR, jx,jy,jz):
 * out 5 per item. op 4 pt_viscosity (:75-80) T -> mu, op 5 pt_conductivity (:83-85)
 * mu -> lam: out 1. Replaces the array-level wrappers' numba point calls
 * (euler_flux, viscous_flux, riemann_flux, split_flux_twopoint, :288-383). */
int hdg_point_eval(const hdg_params* p, int32_t op, int32_t solver, int32_t n, const double* in,
                   double* out, void* stream);
/* testcases.mms_source / k_mms_source (src/testcases.py:51-70): out (n,5) += S(x, t) */
int hdg_mms_source(const hdg_params* p, int32_t n, const double* x, double t, double* out,
                   void* stream);
/* Domain.lift_fill / lift_volume / lift_finish (src/operator.py:667-685):
 * k_lift_fill on the listed sides (d->UL, d->UR -> d->vstar); k_lift_volume
 * (d->g = weak volume term of the prims of U); k_lift_surf_and_jac +
 * k_viscous_contravariant (d->g += surface term, *= 1/J; d->Fvis if set). */
int hdg_lift_fill(const hdg_domain* d, const hdg_params* p, const int32_t* sides, int32_t nsides,
                  void* stream);
int hdg_lift_volume(const hdg_domain* d, const hdg_params* p, const double* U, void* stream);
int hdg_lift_finish(const hdg_domain* d, const hdg_params* p, const double* U, void* stream);
/* Diagnostics: the element pass's per-phase cycle sums (thread 0 of every CTA, top /
 * P1 prims / P2+P3 lifting / P4 volume integral / P5 sum) since the last call, then
 * reset; returns -1 (zeros) unless the library was built with -DE2_TIMING. */
int hdg_debug_phase_cycles(int exact, uint64_t* out8);

#ifdef __cplusplus
}
#endif
#endif /* HEXDG_B200_H */
