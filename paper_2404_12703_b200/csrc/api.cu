// extern "C" boundary of libhexdg_b200.so (declared in include/hexdg_b200.h).
// Thin: validates arguments, picks the exact (-fmad=false) or fast kernel set,
// launches on the caller's stream. No allocation, no synchronisation.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <cuda.h>
#include "common.cuh"

#define HDG_DECLARE_SET(NS)                                                                     \
  namespace NS {                                                                                \
  struct VolArgs {                                                                              \
    double* U;                                                                                  \
    double* out;                                                                                \
    const double* time;                                                                         \
    double t_host, A, B, c;                                                                     \
    int mode;                                                                                   \
  };                                                                                            \
  int run_flux(const hdg_domain&, const hdg_params&, const double*, const int32_t*, int, int,  \
               int, cudaStream_t, const hdg::Gate* = nullptr);                                  \
  int run_lift(const hdg_domain&, const hdg_params&, const double*, cudaStream_t);              \
  int run_elem(const hdg_domain&, const hdg_params&, const double*, const int32_t*, int, bool,  \
               cudaStream_t, const hdg::Gate* = nullptr);                                       \
  int run_update(const hdg_domain&, const hdg_params&, const VolArgs&, const int32_t*, int,    \
                 bool, cudaStream_t, const hdg::Gate* = nullptr);                               \
  int run_volume(const hdg_domain&, const hdg_params&, const VolArgs&, cudaStream_t);           \
  int run_prolong(const hdg_domain&, const double*, const int32_t*, int, cudaStream_t);         \
  int run_bc_traces(const hdg_domain&, const int32_t*, int, cudaStream_t);                      \
  int run_dt(const hdg_domain&, const hdg_params&, const double*, double, double, cudaStream_t); \
  int run_surf_int(const hdg_domain&, const double*, double*, cudaStream_t);                    \
  int run_apply_jac(const hdg_domain&, double*, cudaStream_t);                                  \
  int run_cons_to_prim(const hdg_domain&, const hdg_params&, const double*, double*,            \
                       cudaStream_t);                                                           \
  int run_pack_traces(const hdg_domain&, const double*, const int32_t*, int, double*,           \
                      cudaStream_t);                                                            \
  int run_analysis(const hdg_domain&, const hdg_params&, const double*, const double*, double,  \
                   double*, cudaStream_t);                                                      \
  int run_point(const hdg_params&, int, int, int, const double*, double*, cudaStream_t);      \
  int read_phase_cycles(unsigned long long*);                                                 \
  int run_mms_points(const hdg_params&, int, const double*, double, double*, cudaStream_t);   \
  int run_lift_split(const hdg_domain&, const hdg_params&, int, const double*, const int32_t*, \
                     int, cudaStream_t);                                                        \
  int run_peer_traces(const hdg_domain&, const double*, const int32_t*, const int32_t*,          \
                      const int32_t*, int, const unsigned long long*, const unsigned long long*,  \
                      int, unsigned*, unsigned long long*, cudaStream_t);                        \
  }

HDG_DECLARE_SET(hdg_exact)
HDG_DECLARE_SET(hdg_fast)

namespace hdg {
static thread_local char g_err[512] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
static unsigned long long g_launches = 0;
void count_launch() { __atomic_add_fetch(&g_launches, 1ull, __ATOMIC_RELAXED); }
}  // namespace hdg

extern "C" int64_t hdg_launch_count(void) {
  return (int64_t)__atomic_load_n(&hdg::g_launches, __ATOMIC_RELAXED);
}

static int launched(const char* what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    hdg::set_error("%s: %s", what, cudaGetErrorString(err));
    return -4;
  }
  hdg::count_launch();
  return 0;
}

using hdg::set_error;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define CHECK_PTR(p, name)                                 \
  if (!(p)) {                                              \
    set_error("hexdg_b200: required pointer %s is NULL", name); \
    return -1;                                             \
  }

extern "C" {

int hdg_abi_version(void) { return HDG_ABI_VERSION; }
int64_t hdg_sizeof_domain(void) { return (int64_t)sizeof(hdg_domain); }
int64_t hdg_sizeof_params(void) { return (int64_t)sizeof(hdg_params); }
const char* hdg_last_error(void) { return hdg::g_err; }

int hdg_check_domain(const hdg_domain* d, const hdg_params* p) {
  CHECK_PTR(d, "domain");
  CHECK_PTR(p, "params");
  if (d->N < 1 || d->N > 7) {
    set_error("hexdg_b200: degree N=%d unsupported (1..7)", d->N);
    return -2;
  }
  if (d->ne < 0 || d->ns < 0) {
    set_error("hexdg_b200: negative sizes");
    return -2;
  }
  CHECK_PTR(d->basis, "basis");
  CHECK_PTR(d->Ja, "Ja");
  CHECK_PTR(d->invJ, "invJ");
  CHECK_PTR(d->nvec, "nvec");
  CHECK_PTR(d->ssurf, "ssurf");
  CHECK_PTR(d->ef_info, "ef_info");
  CHECK_PTR(d->side_info, "side_info");
  CHECK_PTR(d->bc_states, "bc_states");
  CHECK_PTR(d->fstar, "fstar");
  CHECK_PTR(d->status, "status");
  if (d->node_type == 0) CHECK_PTR(d->work, "work");
  if (p->viscous) {
    CHECK_PTR(d->fvface, "fvface");
    if (d->node_type == 0) {
      CHECK_PTR(d->vol, "vol");
    } else {
      CHECK_PTR(d->Fvis, "Fvis");
    }
  }
  if (p->shock) {
    CHECK_PTR(d->alpha, "alpha");
    CHECK_PTR(d->fvm0, "fvm0");
    CHECK_PTR(d->fvm1, "fvm1");
    CHECK_PTR(d->fvm2, "fvm2");
    if (d->node_type != 0) {
      set_error("hexdg_b200: shock capturing requires LGL nodes");
      return -2;
    }
  }
  if (p->split && d->node_type != 0) {
    set_error("hexdg_b200: split form requires LGL nodes");
    return -2;
  }
  if (p->source) CHECK_PTR(d->x, "x");
  if (d->node_type != 0) {
    CHECK_PTR(d->UL, "UL");
    CHECK_PTR(d->UR, "UR");
  }
  return 0;
}

#define SET(p) ((p)->exact)
#define HDG_STAGE_NEXT_DT_FLAG 64   /* mode flag bit (<< 4) of the folded next-step dt */

int hdg_phase_lift(const hdg_domain* d, const hdg_params* p, const double* U, void* stream) {
  CHECK_PTR(U, "U");
  return SET(p) ? hdg_exact::run_lift(*d, *p, U, S(stream)) : hdg_fast::run_lift(*d, *p, U, S(stream));
}

int hdg_phase_elem(const hdg_domain* d, const hdg_params* p, const double* U, void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(d->vol, "vol");
  if (d->node_type != 0) {
    set_error("hexdg_b200: hdg_phase_elem needs LGL nodes");
    return -2;
  }
  return SET(p) ? hdg_exact::run_elem(*d, *p, U, nullptr, -1, true, S(stream))
                : hdg_fast::run_elem(*d, *p, U, nullptr, -1, true, S(stream));
}

int hdg_phase_elem_list(const hdg_domain* d, const hdg_params* p, const double* U,
                        const int32_t* elems, int32_t n, int reset_fv, void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(d->vol, "vol");
  if (n > 0) CHECK_PTR(elems, "elems");   // an empty pass still resets the FV count
  if (d->node_type != 0) {
    set_error("hexdg_b200: hdg_phase_elem needs LGL nodes");
    return -2;
  }
  return SET(p) ? hdg_exact::run_elem(*d, *p, U, elems, n, reset_fv != 0, S(stream))
                : hdg_fast::run_elem(*d, *p, U, elems, n, reset_fv != 0, S(stream));
}

static bool make_gate(const hdg_domain* d, const hdg_gate* g, hdg::Gate* out) {
  if (!g || g->n <= 0) {
    *out = hdg::Gate{nullptr, nullptr, 0, 0, nullptr, nullptr};
    return true;
  }
  if (!g->flags || !g->idx || !g->epoch || !d->status) {
    set_error("hexdg_b200: gate needs flags, idx, epoch and the domain status words");
    return false;
  }
  *out = hdg::Gate{reinterpret_cast<const unsigned long long*>(g->flags), g->idx, g->n, g->pos,
                   reinterpret_cast<const unsigned long long*>(g->epoch), d->status};
  return true;
}

int hdg_phase_elem_gated(const hdg_domain* d, const hdg_params* p, const double* U,
                         const int32_t* elems, int32_t n, int reset_fv, const hdg_gate* gate,
                         void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(d->vol, "vol");
  if (n > 0) CHECK_PTR(elems, "elems");
  if (d->node_type != 0) {
    set_error("hexdg_b200: hdg_phase_elem needs LGL nodes");
    return -2;
  }
  hdg::Gate G;
  if (!make_gate(d, gate, &G)) return -1;
  return SET(p) ? hdg_exact::run_elem(*d, *p, U, elems, n, reset_fv != 0, S(stream), &G)
                : hdg_fast::run_elem(*d, *p, U, elems, n, reset_fv != 0, S(stream), &G);
}

int hdg_phase_flux_gated(const hdg_domain* d, const hdg_params* p, const double* U,
                         const int32_t* sides, int32_t nsides, int32_t solver, const hdg_gate* gate,
                         void* stream) {
  if (nsides > 0) CHECK_PTR(sides, "sides");
  hdg::Gate G;
  if (!make_gate(d, gate, &G)) return -1;
  return SET(p) ? hdg_exact::run_flux(*d, *p, U, sides, nsides, solver, 0, S(stream), &G)
                : hdg_fast::run_flux(*d, *p, U, sides, nsides, solver, 0, S(stream), &G);
}

int hdg_phase_update_gated(const hdg_domain* d, const hdg_params* p, double* U, double* out,
                           const double* time_dev, double t_host, double A, double B, double c,
                           int mode, const int32_t* elems, int32_t n, int do_fv,
                           const hdg_gate* gate, void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(out, "Ut/dU");
  CHECK_PTR(d->vol, "vol");
  if (n > 0) CHECK_PTR(elems, "elems");
  if ((mode & 15) != HDG_MODE_STORE_UT) CHECK_PTR(time_dev, "time_dev");
  hdg::Gate G;
  if (!make_gate(d, gate, &G)) return -1;
  if (p->exact) {
    hdg_exact::VolArgs v{U, out, time_dev, t_host, A, B, c, mode};
    return hdg_exact::run_update(*d, *p, v, elems, n, do_fv != 0, S(stream), &G);
  }
  hdg_fast::VolArgs v{U, out, time_dev, t_host, A, B, c, mode};
  return hdg_fast::run_update(*d, *p, v, elems, n, do_fv != 0, S(stream), &G);
}

int hdg_phase_update(const hdg_domain* d, const hdg_params* p, double* U, double* out,
                     const double* time_dev, double t_host, double A, double B, double c, int mode,
                     void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(out, "Ut/dU");
  CHECK_PTR(d->vol, "vol");
  if ((mode & 15) != HDG_MODE_STORE_UT) CHECK_PTR(time_dev, "time_dev");
  if (p->exact) {
    hdg_exact::VolArgs v{U, out, time_dev, t_host, A, B, c, mode};
    return hdg_exact::run_update(*d, *p, v, nullptr, -1, true, S(stream));
  }
  hdg_fast::VolArgs v{U, out, time_dev, t_host, A, B, c, mode};
  return hdg_fast::run_update(*d, *p, v, nullptr, -1, true, S(stream));
}

int hdg_phase_update_list(const hdg_domain* d, const hdg_params* p, double* U, double* out,
                          const double* time_dev, double t_host, double A, double B, double c,
                          int mode, const int32_t* elems, int32_t n, int do_fv, void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(out, "Ut/dU");
  CHECK_PTR(d->vol, "vol");
  if (n > 0) CHECK_PTR(elems, "elems");
  if ((mode & 15) != HDG_MODE_STORE_UT) CHECK_PTR(time_dev, "time_dev");
  if (p->exact) {
    hdg_exact::VolArgs v{U, out, time_dev, t_host, A, B, c, mode};
    return hdg_exact::run_update(*d, *p, v, elems, n, do_fv != 0, S(stream));
  }
  hdg_fast::VolArgs v{U, out, time_dev, t_host, A, B, c, mode};
  return hdg_fast::run_update(*d, *p, v, elems, n, do_fv != 0, S(stream));
}

int hdg_phase_flux(const hdg_domain* d, const hdg_params* p, const double* U, const int32_t* sides,
                   int32_t nsides, int32_t solver, void* stream) {
  if (nsides <= 0) return 0;
  if (!sides && nsides != d->ns) {   // NULL = every local side, in order
    set_error("hexdg_b200: sides == NULL means all %d local sides (got nsides=%d)", d->ns, nsides);
    return -1;
  }
  return SET(p) ? hdg_exact::run_flux(*d, *p, U, sides, nsides, solver, 0, S(stream))
                : hdg_fast::run_flux(*d, *p, U, sides, nsides, solver, 0, S(stream));
}

int hdg_fill_flux_traces(const hdg_domain* d, const hdg_params* p, const int32_t* sides,
                         int32_t nsides, int32_t solver, void* stream) {
  if (nsides <= 0) return 0;
  if (!sides && nsides != d->ns) {
    set_error("hexdg_b200: sides == NULL means all %d local sides (got nsides=%d)", d->ns, nsides);
    return -1;
  }
  CHECK_PTR(d->UL, "UL");
  CHECK_PTR(d->UR, "UR");
  return SET(p) ? hdg_exact::run_flux(*d, *p, nullptr, sides, nsides, solver, 1, S(stream))
                : hdg_fast::run_flux(*d, *p, nullptr, sides, nsides, solver, 1, S(stream));
}

int hdg_phase_volume(const hdg_domain* d, const hdg_params* p, double* U, double* out,
                     const double* time_dev, double t_host, double A, double B, double c, int mode,
                     void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(out, "Ut/dU");
  if ((mode & 15) != HDG_MODE_STORE_UT) CHECK_PTR(time_dev, "time_dev");
  // the fused element pass has no dt epilogue: a folded next-step dt is its own pass
  // over the updated U
  const int dtflag = (HDG_STAGE_NEXT_DT_FLAG << 4);
  const bool next_dt = (mode & dtflag) && (mode & 15) != HDG_MODE_STORE_UT;
  mode &= ~dtflag;
  int rc;
  if (p->exact) {
    hdg_exact::VolArgs v{U, out, time_dev, t_host, A, B, c, mode};
    rc = hdg_exact::run_volume(*d, *p, v, S(stream));
  } else {
    hdg_fast::VolArgs v{U, out, time_dev, t_host, A, B, c, mode};
    rc = hdg_fast::run_volume(*d, *p, v, S(stream));
  }
  if (rc || !next_dt) return rc;
  return hdg_local_dt(d, p, U, p->cfl, p->cfl_visc, stream);
}

// the full single-rank stage: [lift] -> flux(all local sides) -> volume
static int stage_impl(const hdg_domain* d, const hdg_params* p, double* U, double* out,
                      const double* time_dev, double t_host, double A, double B, double c, int mode,
                      const int32_t* sides, int nsides, void* stream) {
  int rc = hdg_check_domain(d, p);
  if (rc) return rc;
  if (d->node_type != 0) {
    set_error("hexdg_b200: fused stage needs LGL (use prolong + phases for GL)");
    return -2;
  }
  if (p->viscous || (d->vol && !p->shock)) {
    // A (lifting + volume, TMA-pipelined) -> surface fluxes -> C (surface + update);
    // Euler with shock capturing keeps the single fused element pass below
    if ((rc = hdg_phase_elem(d, p, U, stream))) return rc;
    if ((rc = hdg_phase_flux(d, p, U, sides, nsides, p->surf_solver, stream))) return rc;
    return hdg_phase_update(d, p, U, out, time_dev, t_host, A, B, c, mode, stream);
  }
  // Euler: surface fluxes -> one fused element pass
  if ((rc = hdg_phase_flux(d, p, U, sides, nsides, p->surf_solver, stream))) return rc;
  return hdg_phase_volume(d, p, U, out, time_dev, t_host, A, B, c, mode, stream);
}

int hdg_rhs(const hdg_domain* d, const hdg_params* p, const double* U, double* Ut, double t,
                  const int32_t* sides, int32_t nsides, void* stream) {
  return stage_impl(d, p, const_cast<double*>(U), Ut, nullptr, t, 0.0, 0.0, 0.0,
                    HDG_MODE_STORE_UT, sides, nsides, stream);
}

int hdg_stage(const hdg_domain* d, const hdg_params* p, double* U, double* dU,
                    const double* time_dev, double A, double B, double c, int first,
                    const int32_t* sides, int32_t nsides, void* stream) {
  const int mode = ((first & 1) ? HDG_MODE_LSERK_FIRST : HDG_MODE_LSERK) |
                   ((first & HDG_STAGE_NEXT_DT) ? (HDG_STAGE_NEXT_DT_FLAG << 4) : 0);
  return stage_impl(d, p, U, dU, time_dev, 0.0, A, B, c, mode, sides, nsides, stream);
}

int hdg_cons_to_prim(const hdg_domain* d, const hdg_params* p, const double* U, double* prim,
                     void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(prim, "prim");
  return SET(p) ? hdg_exact::run_cons_to_prim(*d, *p, U, prim, S(stream))
                : hdg_fast::run_cons_to_prim(*d, *p, U, prim, S(stream));
}

int hdg_prolong(const hdg_domain* d, const double* U, const int32_t* rows, int32_t nrows,
                void* stream) {
  if (nrows <= 0) return 0;
  CHECK_PTR(rows, "rows");
  CHECK_PTR(d->UL, "UL");
  return hdg_exact::run_prolong(*d, U, rows, nrows, S(stream));
}

int hdg_apply_bc_traces(const hdg_domain* d, const int32_t* sides, int32_t nsides, void* stream) {
  if (nsides <= 0) return 0;
  CHECK_PTR(d->UR, "UR");
  return hdg_exact::run_bc_traces(*d, sides, nsides, S(stream));
}

int hdg_surf_int(const hdg_domain* d, const double* fstar, double* Ut, void* stream) {
  CHECK_PTR(fstar, "fstar");
  CHECK_PTR(Ut, "Ut");
  return hdg_exact::run_surf_int(*d, fstar, Ut, S(stream));
}

int hdg_apply_jac(const hdg_domain* d, double* Ut, void* stream) {
  CHECK_PTR(Ut, "Ut");
  CHECK_PTR(d->J, "J");
  return hdg_exact::run_apply_jac(*d, Ut, S(stream));
}

int hdg_local_dt(const hdg_domain* d, const hdg_params* p, const double* U, double cfl,
                 double cfl_visc, void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(d->J, "J");
  CHECK_PTR(d->dt_bits, "dt_bits");
  return SET(p) ? hdg_exact::run_dt(*d, *p, U, cfl, cfl_visc, S(stream))
                : hdg_fast::run_dt(*d, *p, U, cfl, cfl_visc, S(stream));
}

int hdg_analysis_partials(const hdg_domain* d, const hdg_params* p, const double* U,
                          const double* g, double mu0, double* out, void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(out, "out");
  CHECK_PTR(d->J, "J");
  if (p->viscous) CHECK_PTR(g, "g");
  if (!(mu0 > 0.0)) {
    set_error("hexdg_b200: mu0 must be positive (pass 1.0 when there is no reference viscosity)");
    return -1;
  }
  return SET(p) ? hdg_exact::run_analysis(*d, *p, U, g, mu0, out, S(stream))
                : hdg_fast::run_analysis(*d, *p, U, g, mu0, out, S(stream));
}

}  // extern "C"

// ---------------------------------------------------------------------------
// generic helpers (precision-neutral)

__global__ void lserk_kernel(double* __restrict__ U, double* __restrict__ dU,
                             const double* __restrict__ Ut, long n, double A, double B, double dt,
                             int first) {
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long)gridDim.x * blockDim.x) {
    const double du = first ? __dmul_rn(dt, Ut[t]) : __dadd_rn(__dmul_rn(dU[t], A), __dmul_rn(dt, Ut[t]));
    dU[t] = du;
    U[t] = __dadd_rn(U[t], __dmul_rn(B, du));
  }
}

__global__ void pack_kernel(const double* __restrict__ src, const int32_t* __restrict__ idx,
                            long n, int width, double* __restrict__ buf) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * width) return;
  const long k = t / width;
  buf[t] = src[(long)idx[k] * width + (t % width)];
}

__global__ void unpack_kernel(const double* __restrict__ buf, const int32_t* __restrict__ idx,
                              long n, int width, double* __restrict__ dst) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * width) return;
  const long k = t / width;
  dst[(long)idx[k] * width + (t % width)] = buf[t];
}

// rows of a local array straight into the neighbours' arrays (see peer_send_traces_kernel)
__global__ void __launch_bounds__(256) peer_send_rows_kernel(
    const double* __restrict__ src_rows, int width, const int32_t* __restrict__ nbr,
    const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int n,
    const unsigned long long* __restrict__ dst_base, const unsigned long long* __restrict__ flag_ptrs,
    int n_nbr, unsigned* counter, unsigned long long* epoch) {
  // grid-stride over the words (at most a few blocks per SM: every block pays one
  // system-scope fence and one counter atomic in publish_epoch)
  const long total = (long)n * width;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const int k = (int)(t / width), j = (int)(t % width);
    reinterpret_cast<double*>(dst_base[nbr[k]])[(size_t)dst[k] * width + j] =
        src_rows[(size_t)src[k] * width + j];
  }
  hdg::publish_epoch(counter, flag_ptrs, n_nbr, epoch);
}

// one thread per neighbour: bounded acquire-spin until the flag word reaches the
// epoch this rank's own send of the phase (always issued first) wrote to its send
// counter -- every rank sends each phase equally often; a stuck peer sets
// HDG_STATUS_PEER_TIMEOUT after ~10 s instead of hanging the GPU
__global__ void peer_wait_kernel(const unsigned long long* flags, const int32_t* idx, int n,
                                 const unsigned long long* epoch_ctr, int32_t* status) {
  if ((int)threadIdx.x >= n) return;
  const unsigned long long epoch = *reinterpret_cast<const volatile unsigned long long*>(epoch_ctr);
  const unsigned long long* f = flags + idx[threadIdx.x];
  const long long t0 = clock64();
  while (hdg::ld_acquire_sys_u64(f) < epoch) {
    __nanosleep(256);
    if (clock64() - t0 > 20000000000LL) {
      atomicExch(&status[HDG_STATUS_PEER_TIMEOUT], 1);
      break;
    }
  }
}

// min of the dt bit patterns and max of the status words over all ranks through
// peer memory (the NCCL all-reduce of _compute_dt, src/parallel.py:567-579):
// thread q stores this rank's values into rank q's slot array (parity of the
// epoch, so a rank one step ahead never overwrites values still being read),
// releases the epoch into rank q's flag word, then waits for rank q's flag
__global__ void peer_allreduce_kernel(unsigned long long* dt_bits, int32_t* status,
                                      const unsigned long long* slot_ptrs,
                                      const unsigned long long* flag_ptrs,
                                      const long long* my_slots, const unsigned long long* my_flags,
                                      int me, int world, unsigned long long* epoch_ctr) {
  constexpr int W = 10;   // dt bits + 8 status words + pad
  __shared__ unsigned long long s_epoch;
  __shared__ int s_timeout;
  if (threadIdx.x == 0) {
    s_epoch = atomicAdd(epoch_ctr, 1ull) + 1ull;
    s_timeout = 0;
  }
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  const int par = (int)(epoch & 1ull);
  const int q = threadIdx.x;
  if (q < world) {
    long long* dst = reinterpret_cast<long long*>(slot_ptrs[q]) + ((size_t)par * world + me) * W;
    dst[0] = (long long)dt_bits[0];
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[1 + i] = status[i];
    __threadfence_system();
    hdg::st_release_sys_u64(reinterpret_cast<unsigned long long*>(flag_ptrs[q]) + me, epoch);
    const long long t0 = clock64();
    while (hdg::ld_acquire_sys_u64(my_flags + q) < epoch) {
      __nanosleep(128);
      if (clock64() - t0 > 20000000000LL) {
        s_timeout = 1;
        break;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long best = 0xFFFFFFFFFFFFFFFFull;
    int st[8];
    for (int i = 0; i < 8; ++i) st[i] = INT32_MIN;
    for (int r = 0; r < world; ++r) {
      const long long* v = my_slots + ((size_t)par * world + r) * W;
      const unsigned long long b = (unsigned long long)v[0];
      best = b < best ? b : best;
      for (int i = 0; i < 8; ++i) st[i] = (int)v[1 + i] > st[i] ? (int)v[1 + i] : st[i];
    }
    dt_bits[0] = best;
    for (int i = 0; i < 8; ++i) status[i] = st[i];
    if (s_timeout) status[HDG_STATUS_PEER_TIMEOUT] = 1;
  }
}

__global__ void dt_finalize_kernel(unsigned long long* dt_bits, double* time, double tend) {
  double dt = __longlong_as_double((long long)dt_bits[0]);
  if (time[0] + dt > tend) dt = tend - time[0];
  time[1] = dt;
  dt_bits[0] = 0x7ff0000000000000ULL;   // +inf: the next (folded) local-dt accumulation
}

__global__ void time_advance_kernel(double* time) { time[0] = time[0] + time[1]; }

extern "C" {

int hdg_lserk_update(double* U, double* dU, const double* Ut, int64_t n, double A, double B,
                     double dt, int first, void* stream) {
  CHECK_PTR(U, "U");
  CHECK_PTR(dU, "dU");
  CHECK_PTR(Ut, "Ut");
  if (n <= 0) return 0;
  long blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  lserk_kernel<<<(int)blocks, 256, 0, S(stream)>>>(U, dU, Ut, n, A, B, dt, first);
  return launched("lserk_kernel");
}

int hdg_pack(const double* src, const int32_t* idx, int32_t n, int32_t width, double* buf,
             void* stream) {
  if (n <= 0) return 0;
  const long total = (long)n * width;
  pack_kernel<<<(int)((total + 255) / 256), 256, 0, S(stream)>>>(src, idx, n, width, buf);
  return launched("pack_kernel");
}

int hdg_pack_traces(const hdg_domain* d, const double* U, const int32_t* sides, int32_t n,
                    double* buf, void* stream) {
  if (n <= 0) return 0;
  CHECK_PTR(sides, "sides");
  CHECK_PTR(buf, "buf");
  return hdg_exact::run_pack_traces(*d, U, sides, n, buf, S(stream));
}

int hdg_peer_send_traces(const hdg_domain* d, const double* U, const int32_t* nbr,
                         const int32_t* src, const int32_t* dst, int32_t n, const uint64_t* dst_base,
                         const uint64_t* flag_ptrs, int32_t n_nbr, uint32_t* counter,
                         uint64_t* epoch, void* stream) {
  if (n_nbr <= 0) return 0;
  CHECK_PTR(U, "U");
  CHECK_PTR(dst_base, "dst_base");
  CHECK_PTR(flag_ptrs, "flag_ptrs");
  CHECK_PTR(counter, "counter");
  if (n > 0) {
    CHECK_PTR(nbr, "nbr");
    CHECK_PTR(src, "src");
    CHECK_PTR(dst, "dst");
  }
  if (n_nbr > 256) {
    set_error("hexdg_b200: at most 256 neighbours");
    return -1;
  }
  return hdg_exact::run_peer_traces(*d, U, nbr, src, dst, n,
                                    reinterpret_cast<const unsigned long long*>(dst_base),
                                    reinterpret_cast<const unsigned long long*>(flag_ptrs), n_nbr,
                                    counter, reinterpret_cast<unsigned long long*>(epoch),
                                    S(stream));
}

int hdg_peer_send_rows(const double* src_rows, int32_t width, const int32_t* nbr,
                       const int32_t* src, const int32_t* dst, int32_t n, const uint64_t* dst_base,
                       const uint64_t* flag_ptrs, int32_t n_nbr, uint32_t* counter,
                       uint64_t* epoch, void* stream) {
  if (n_nbr <= 0) return 0;
  CHECK_PTR(src_rows, "src_rows");
  CHECK_PTR(dst_base, "dst_base");
  CHECK_PTR(flag_ptrs, "flag_ptrs");
  CHECK_PTR(counter, "counter");
  if (n > 0) {
    CHECK_PTR(nbr, "nbr");
    CHECK_PTR(src, "src");
    CHECK_PTR(dst, "dst");
  }
  if (n_nbr > 256) {
    set_error("hexdg_b200: at most 256 neighbours");
    return -1;
  }
  const long total = (long)n * width;
  const long want = total > 0 ? (total + 255) / 256 : 1, cap = 2L * hdg::sm_count();
  const int blocks = (int)(want < cap ? want : cap);
  peer_send_rows_kernel<<<blocks, 256, 0, S(stream)>>>(
      src_rows, width, nbr, src, dst, n, reinterpret_cast<const unsigned long long*>(dst_base),
      reinterpret_cast<const unsigned long long*>(flag_ptrs), n_nbr, counter,
      reinterpret_cast<unsigned long long*>(epoch));
  return launched("peer_send_rows_kernel");
}

int hdg_ipc_export(const void* ptr, void* handle, int64_t* offset) {
  CHECK_PTR(ptr, "ptr");
  CHECK_PTR(handle, "handle");
  CHECK_PTR(offset, "offset");
  // allocation base through the driver entry point (the library links only cudart)
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        !fn) {
      set_error("cudaGetDriverEntryPoint(cuMemGetAddressRange) failed");
      return -4;
    }
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) {
    set_error("cuMemGetAddressRange failed");
    return -4;
  }
  cudaIpcMemHandle_t h;
  cudaError_t err = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (err != cudaSuccess) {
    set_error("cudaIpcGetMemHandle: %s", cudaGetErrorString(err));
    return -4;
  }
  memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return 0;
}

int hdg_ipc_open(const void* handle, void** ptr) {
  CHECK_PTR(handle, "handle");
  CHECK_PTR(ptr, "ptr");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t err = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (err != cudaSuccess) {
    set_error("cudaIpcOpenMemHandle: %s", cudaGetErrorString(err));
    return -4;
  }
  return 0;
}

int hdg_ipc_close(void* ptr) {
  cudaError_t err = cudaIpcCloseMemHandle(ptr);
  if (err != cudaSuccess) {
    set_error("cudaIpcCloseMemHandle: %s", cudaGetErrorString(err));
    return -4;
  }
  return 0;
}

int hdg_peer_wait(const uint64_t* flags, const int32_t* idx, int32_t n, const uint64_t* epoch,
                  int32_t* status, void* stream) {
  if (n <= 0) return 0;
  CHECK_PTR(flags, "flags");
  CHECK_PTR(idx, "idx");
  CHECK_PTR(epoch, "epoch");
  CHECK_PTR(status, "status");
  if (n > 1024) {
    set_error("hexdg_b200: at most 1024 flags per wait");
    return -1;
  }
  peer_wait_kernel<<<1, ((n + 31) / 32) * 32, 0, S(stream)>>>(
      reinterpret_cast<const unsigned long long*>(flags), idx, n,
      reinterpret_cast<const unsigned long long*>(epoch), status);
  return launched("peer_wait_kernel");
}

int hdg_peer_allreduce_dt(const hdg_domain* d, const uint64_t* slot_ptrs, const uint64_t* flag_ptrs,
                          const int64_t* my_slots, const uint64_t* my_flags, int32_t me,
                          int32_t world, uint64_t* epoch, void* stream) {
  CHECK_PTR(d->dt_bits, "dt_bits");
  CHECK_PTR(d->status, "status");
  CHECK_PTR(slot_ptrs, "slot_ptrs");
  CHECK_PTR(flag_ptrs, "flag_ptrs");
  CHECK_PTR(my_slots, "my_slots");
  CHECK_PTR(my_flags, "my_flags");
  CHECK_PTR(epoch, "epoch");
  if (world < 1 || world > 32 || me < 0 || me >= world) {
    set_error("hexdg_b200: peer all-reduce needs 1 <= world <= 32");
    return -1;
  }
  peer_allreduce_kernel<<<1, 32, 0, S(stream)>>>(
      reinterpret_cast<unsigned long long*>(d->dt_bits), d->status,
      reinterpret_cast<const unsigned long long*>(slot_ptrs),
      reinterpret_cast<const unsigned long long*>(flag_ptrs),
      reinterpret_cast<const long long*>(my_slots),
      reinterpret_cast<const unsigned long long*>(my_flags), me, world,
      reinterpret_cast<unsigned long long*>(epoch));
  return launched("peer_allreduce_kernel");
}

int hdg_unpack(const double* buf, const int32_t* idx, int32_t n, int32_t width, double* dst,
               void* stream) {
  if (n <= 0) return 0;
  const long total = (long)n * width;
  unpack_kernel<<<(int)((total + 255) / 256), 256, 0, S(stream)>>>(buf, idx, n, width, dst);
  return launched("unpack_kernel");
}

int hdg_dt_finalize(const hdg_domain* d, double* time_dev, double tend, void* stream) {
  CHECK_PTR(d->dt_bits, "dt_bits");
  CHECK_PTR(time_dev, "time_dev");
  dt_finalize_kernel<<<1, 1, 0, S(stream)>>>(reinterpret_cast<unsigned long long*>(d->dt_bits),
                                             time_dev, tend);
  return launched("dt_finalize_kernel");
}

int hdg_time_advance(double* time_dev, void* stream) {
  CHECK_PTR(time_dev, "time_dev");
  time_advance_kernel<<<1, 1, 0, S(stream)>>>(time_dev);
  return launched("time_advance_kernel");
}

}  // extern "C"

/* ---- API-granularity calls (api_kernels.cuh) ------------------------------ */
int hdg_point_eval(const hdg_params* p, int32_t op, int32_t solver, int32_t n, const double* in,
                   double* out, void* stream) {
  CHECK_PTR(p, "params");
  if (n > 0) {
    CHECK_PTR(in, "in");
    CHECK_PTR(out, "out");
  }
  return SET(p) ? hdg_exact::run_point(*p, op, solver, n, in, out, S(stream))
                : hdg_fast::run_point(*p, op, solver, n, in, out, S(stream));
}

int hdg_mms_source(const hdg_params* p, int32_t n, const double* x, double t, double* out,
                   void* stream) {
  CHECK_PTR(p, "params");
  if (n > 0) {
    CHECK_PTR(x, "x");
    CHECK_PTR(out, "out");
  }
  return SET(p) ? hdg_exact::run_mms_points(*p, n, x, t, out, S(stream))
                : hdg_fast::run_mms_points(*p, n, x, t, out, S(stream));
}

int hdg_lift_fill(const hdg_domain* d, const hdg_params* p, const int32_t* sides, int32_t nsides,
                  void* stream) {
  CHECK_PTR(d, "domain");
  CHECK_PTR(p, "params");
  CHECK_PTR(d->UL, "UL");
  CHECK_PTR(d->UR, "UR");
  CHECK_PTR(d->vstar, "vstar");
  if (nsides > 0) CHECK_PTR(sides, "sides");
  return SET(p) ? hdg_exact::run_lift_split(*d, *p, 0, nullptr, sides, nsides, S(stream))
                : hdg_fast::run_lift_split(*d, *p, 0, nullptr, sides, nsides, S(stream));
}

int hdg_lift_volume(const hdg_domain* d, const hdg_params* p, const double* U, void* stream) {
  CHECK_PTR(d, "domain");
  CHECK_PTR(p, "params");
  CHECK_PTR(U, "U");
  CHECK_PTR(d->g, "g");
  return SET(p) ? hdg_exact::run_lift_split(*d, *p, 1, U, nullptr, 0, S(stream))
                : hdg_fast::run_lift_split(*d, *p, 1, U, nullptr, 0, S(stream));
}

int hdg_lift_finish(const hdg_domain* d, const hdg_params* p, const double* U, void* stream) {
  CHECK_PTR(d, "domain");
  CHECK_PTR(p, "params");
  CHECK_PTR(U, "U");
  CHECK_PTR(d->g, "g");
  CHECK_PTR(d->vstar, "vstar");
  return SET(p) ? hdg_exact::run_lift_split(*d, *p, 2, U, nullptr, 0, S(stream))
                : hdg_fast::run_lift_split(*d, *p, 2, U, nullptr, 0, S(stream));
}

/* E2_TIMING builds: the element kernel's per-phase cycle sums (read + reset) */
extern "C" int hdg_debug_phase_cycles(int exact, uint64_t* out8) {
  CHECK_PTR(out8, "out");
  return exact ? hdg_exact::read_phase_cycles(reinterpret_cast<unsigned long long*>(out8))
               : hdg_fast::read_phase_cycles(reinterpret_cast<unsigned long long*>(out8));
}
