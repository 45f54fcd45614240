// Host-side launchers for one kernel set (included inside hdg_exact / hdg_fast
// after kernels.cuh). Dispatch on the degree N (1..7) and the operator flags.

template <int N, bool LGL>
constexpr size_t lift_smem() {
  using DM = Dim<N>;
  return sizeof(double) * (((DM::BASIS + 1) & ~1) +
                           DM::EPB * (13 * DM::n3 + 24 * DM::n2 + (LGL ? 0 : 12 * DM::n3)));
}

template <int N, bool SPLIT, bool VISC, bool SHOCK>
constexpr size_t volume_smem() {
  using DM = Dim<N>;
  return sizeof(double) *
         (((DM::BASIS + 1) & ~1) + DM::EPB * (7 * DM::n3 + vol_work<N, SPLIT, VISC, SHOCK>()));
}

template <typename K>
static int prep_kernel(K kernel, size_t smem) {
  // opt in above the default 48 KB with margin: the kernels' static shared memory
  // (barriers, face tables, reductions) counts against the same limit
  if (smem > 40 * 1024) {
    cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
    if (err != cudaSuccess) {
      hdg::set_error("cudaFuncSetAttribute(smem=%zu): %s", smem, cudaGetErrorString(err));
      return -3;
    }
  }
  return 0;
}

static int check_launch(const char* what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    hdg::set_error("%s launch failed: %s", what, cudaGetErrorString(err));
    return -4;
  }
  hdg::count_launch();
  return 0;
}

#define HDG_DISPATCH_N(N_, CALL)                      \
  switch (N_) {                                       \
    case 1: return CALL(1);                           \
    case 2: return CALL(2);                           \
    case 3: return CALL(3);                           \
    case 4: return CALL(4);                           \
    case 5: return CALL(5);                           \
    case 6: return CALL(6);                           \
    case 7: return CALL(7);                           \
    default: hdg::set_error("unsupported degree N=%d (1..7)", (int)N_); return -2; \
  }

// ---- flux ---------------------------------------------------------------
template <int N>
static int flux_n(const hdg_domain& D, const hdg_params& P, const double* U, const int32_t* sides,
                  int nsides, int solver, int from_arrays, const Gate& G, cudaStream_t st) {
  if (nsides <= 0) return 0;
  constexpr int n2 = (N + 1) * (N + 1);
  const long total = (long)nsides * n2;
  const int blocks = (int)((total + 63) / 64);
  const bool lgl = D.node_type == 0;
  const bool visc = P.viscous != 0;
  if (lgl && visc) flux_kernel<N, true, true><<<blocks, 64, 0, st>>>(D, P, U, sides, nsides, solver, from_arrays, G);
  else if (lgl) flux_kernel<N, true, false><<<blocks, 64, 0, st>>>(D, P, U, sides, nsides, solver, from_arrays, G);
  else if (visc) flux_kernel<N, false, true><<<blocks, 64, 0, st>>>(D, P, U, sides, nsides, solver, from_arrays, G);
  else flux_kernel<N, false, false><<<blocks, 64, 0, st>>>(D, P, U, sides, nsides, solver, from_arrays, G);
  return check_launch("flux_kernel");
}

static const Gate kNoGate{nullptr, nullptr, 0, 0, nullptr, nullptr};

int run_flux(const hdg_domain& D, const hdg_params& P, const double* U, const int32_t* sides,
             int nsides, int solver, int from_arrays, cudaStream_t st, const Gate* gate) {
  const Gate& G = gate ? *gate : kNoGate;
#define CALL(n) flux_n<n>(D, P, U, sides, nsides, solver, from_arrays, G, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

// ---- lift ---------------------------------------------------------------
template <int N, bool LGL>
static int lift_nl(const hdg_domain& D, const hdg_params& P, const double* U, cudaStream_t st) {
  using DM = Dim<N>;
  constexpr size_t smem = lift_smem<N, LGL>();
  static int prepared = prep_kernel(lift_kernel<N, LGL>, smem);
  if (prepared) return prepared;
  const int blocks = (D.ne + DM::EPB - 1) / DM::EPB;
  if (blocks == 0) return 0;
  lift_kernel<N, LGL><<<blocks, DM::THREADS, smem, st>>>(D, P, U);
  return check_launch("lift_kernel");
}

template <int N>
static int lift_n(const hdg_domain& D, const hdg_params& P, const double* U, cudaStream_t st) {
  return D.node_type == 0 ? lift_nl<N, true>(D, P, U, st) : lift_nl<N, false>(D, P, U, st);
}

int run_lift(const hdg_domain& D, const hdg_params& P, const double* U, cudaStream_t st) {
#define CALL(n) lift_n<n>(D, P, U, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

// ---- volume -------------------------------------------------------------
template <int N, bool SPLIT, bool VISC, bool SHOCK>
static int volume_nf(const hdg_domain& D, const hdg_params& P, const VolArgs& V, cudaStream_t st) {
  using DM = Dim<N>;
  constexpr size_t smem = volume_smem<N, SPLIT, VISC, SHOCK>();
  static int prepared = prep_kernel(volume_kernel<N, SPLIT, VISC, SHOCK>, smem);
  if (prepared) return prepared;
  const int blocks = (D.ne + DM::EPB - 1) / DM::EPB;
  if (blocks == 0) return 0;
  volume_kernel<N, SPLIT, VISC, SHOCK><<<blocks, DM::THREADS, smem, st>>>(D, P, V);
  return check_launch("volume_kernel");
}

template <int N>
static int volume_n(const hdg_domain& D, const hdg_params& P, const VolArgs& V, cudaStream_t st) {
  const int key = (P.split ? 4 : 0) | (P.viscous ? 2 : 0) | (P.shock ? 1 : 0);
  switch (key) {
    case 0: return volume_nf<N, false, false, false>(D, P, V, st);
    case 1: return volume_nf<N, false, false, true>(D, P, V, st);
    case 2: return volume_nf<N, false, true, false>(D, P, V, st);
    case 3: return volume_nf<N, false, true, true>(D, P, V, st);
    case 4: return volume_nf<N, true, false, false>(D, P, V, st);
    case 5: return volume_nf<N, true, false, true>(D, P, V, st);
    case 6: return volume_nf<N, true, true, false>(D, P, V, st);
    default: return volume_nf<N, true, true, true>(D, P, V, st);
  }
}

int run_volume(const hdg_domain& D, const hdg_params& P, const VolArgs& V, cudaStream_t st) {
#define CALL(n) volume_n<n>(D, P, V, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

// ---- small kernels --------------------------------------------------------
template <int N>
static int prolong_n(const hdg_domain& D, const double* U, const int32_t* rows, int nrows,
                     cudaStream_t st) {
  if (nrows <= 0) return 0;
  constexpr int n2 = (N + 1) * (N + 1);
  const long total = (long)nrows * n2;
  prolong_kernel<N><<<(int)((total + 255) / 256), 256, 0, st>>>(D, U, rows, nrows);
  return check_launch("prolong_kernel");
}

int run_prolong(const hdg_domain& D, const double* U, const int32_t* rows, int nrows,
                cudaStream_t st) {
#define CALL(n) prolong_n<n>(D, U, rows, nrows, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

int run_bc_traces(const hdg_domain& D, const int32_t* sides, int nsides, cudaStream_t st) {
  if (nsides <= 0) return 0;
  const int n2 = (D.N + 1) * (D.N + 1);
  const long total = (long)nsides * n2 * 5;
  bc_traces_kernel<<<(int)((total + 255) / 256), 256, 0, st>>>(D, sides, nsides, n2);
  return check_launch("bc_traces_kernel");
}

template <int N>
static int dt_n(const hdg_domain& D, const hdg_params& P, const double* U, double cfl, double cflv,
                cudaStream_t st) {
  constexpr int n3 = (N + 1) * (N + 1) * (N + 1);
  const long total = (long)D.ne * n3;
  if (total == 0) return 0;
  long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;   // grid-stride: few atomics
  dt_kernel<N><<<(int)blocks, 256, 0, st>>>(D, P, U, cfl, cflv);
  return check_launch("dt_kernel");
}

int run_dt(const hdg_domain& D, const hdg_params& P, const double* U, double cfl, double cflv,
           cudaStream_t st) {
#define CALL(n) dt_n<n>(D, P, U, cfl, cflv, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

template <int N>
static int analysis_n(const hdg_domain& D, const hdg_params& P, const double* U, const double* g,
                      double mu0, double* out, cudaStream_t st) {
  if (D.ne == 0) return 0;
  analysis_kernel<N><<<(D.ne + 127) / 128, 128, 0, st>>>(D, P, U, g, mu0, out);
  return check_launch("analysis_kernel");
}

int run_analysis(const hdg_domain& D, const hdg_params& P, const double* U, const double* g,
                 double mu0, double* out, cudaStream_t st) {
#define CALL(n) analysis_n<n>(D, P, U, g, mu0, out, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

template <int N>
static int surf_int_n(const hdg_domain& D, const double* fstar, double* Ut, cudaStream_t st) {
  constexpr int n3 = (N + 1) * (N + 1) * (N + 1);
  const long total = (long)D.ne * n3;
  if (total == 0) return 0;
  surf_int_kernel<N><<<(int)((total + 255) / 256), 256, 0, st>>>(D, fstar, Ut);
  return check_launch("surf_int_kernel");
}

int run_surf_int(const hdg_domain& D, const double* fstar, double* Ut, cudaStream_t st) {
#define CALL(n) surf_int_n<n>(D, fstar, Ut, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

int run_apply_jac(const hdg_domain& D, double* Ut, cudaStream_t st) {
  const long n = (long)D.ne * (D.N + 1) * (D.N + 1) * (D.N + 1);
  if (n == 0) return 0;
  apply_jac_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(D.J, Ut, n);
  return check_launch("apply_jac_kernel");
}

int run_cons_to_prim(const hdg_domain& D, const hdg_params& P, const double* U, double* prim,
                     cudaStream_t st) {
  const long n = (long)D.ne * (D.N + 1) * (D.N + 1) * (D.N + 1);
  if (n == 0) return 0;
  cons_to_prim_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(D, P, U, prim, n);
  return check_launch("cons_to_prim_kernel");
}

// ---- Navier-Stokes LGL stage split (elem.cuh) ---------------------------------

// Dsplit of the domain's basis into the constant bank the element kernel reads
// (stream-ordered device-to-device copy, graph-capturable; re-issued only when the
// basis pointer changes: LGL Dsplit of a degree is one fixed table)
template <int N>
static int upload_dsplit(const hdg_domain& D, cudaStream_t st) {
  static const double* last = nullptr;
  if (last == D.basis) return 0;
  constexpr int n2 = (N + 1) * (N + 1);
  cudaError_t err = cudaMemcpyToSymbolAsync(c_dsplit, D.basis + Dim<N>::oDsplit,
                                            n2 * sizeof(double),
                                            N * 64 * sizeof(double),
                                            cudaMemcpyDeviceToDevice, st);
  if (err != cudaSuccess) {
    hdg::set_error("cudaMemcpyToSymbolAsync(c_dsplit): %s", cudaGetErrorString(err));
    return -4;
  }
  last = D.basis;
  return 0;
}

template <int N, bool SPLIT, bool VISC>
static int elem_nf(const hdg_domain& D, const hdg_params& P, const double* U, const int32_t* elist,
                   int nlist, const Gate& G, cudaStream_t st) {
  using DM = Dim<N>;
  constexpr size_t smem = elem_smem<N, SPLIT, VISC>();
  static int resident = -1;
  if (resident < 0) {
    int rc = prep_kernel(elem_kernel<N, SPLIT, VISC>, smem);
    if (rc) return rc;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, elem_kernel<N, SPLIT, VISC>, DM::THREADS,
                                                  smem);
    resident = sms * (per > 0 ? per : 1);
  }
  if (elist && DM::EPB != 1) {
    hdg::set_error("element lists need one element per block (N >= 4)");
    return -2;
  }
  const int groups = elist ? nlist : (D.ne + DM::EPB - 1) / DM::EPB;
  if (groups <= 0) return 0;
  // persistent: one block per resident slot (never more blocks than groups)
  const int blocks = groups < resident ? groups : resident;
  elem_kernel<N, SPLIT, VISC><<<blocks, DM::THREADS, smem, st>>>(D, P, U, elist, nlist, G);
  return check_launch("elem_kernel");
}

// two nodes per thread + line-per-thread volume integral (elem2.cuh): both kernel
// sets, split form, N = 5 / 7, Navier-Stokes or shock-free Euler
template <int N>
constexpr bool kElemPair = (N == 7 || N == 5);


template <int N, bool VISC, bool SHOCK, bool LISTED, bool DBG>
static int elem2_kf(const hdg_domain& D, const hdg_params& P, const double* U,
                    const int32_t* elist, int nlist, const Gate& G, cudaStream_t st) {
  using DM = Dim<N>;
  constexpr size_t smem = E2Map<N, VISC>::SMEM;
  if (int rc = upload_dsplit<N>(D, st)) return rc;
  constexpr int threads = elem2_threads<N>();
  static int resident = -1;
  if (resident < 0) {
    int rc = prep_kernel(elem2_kernel<N, VISC, SHOCK, LISTED, DBG>, smem);
    if (rc) return rc;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, elem2_kernel<N, VISC, SHOCK, LISTED, DBG>,
                                                  threads, smem);
    resident = sms * (per > 0 ? per : 1);
  }
  const int groups = elist ? nlist : D.ne;
  if (groups <= 0) return 0;
  const int blocks = groups < resident ? groups : resident;
  elem2_kernel<N, VISC, SHOCK, LISTED, DBG><<<blocks, threads, smem, st>>>(D, P, U, elist, nlist, G);
  return check_launch("elem2_kernel");
}

template <int N, bool VISC, bool SHOCK>
static int elem2_nf(const hdg_domain& D, const hdg_params& P, const double* U,
                    const int32_t* elist, int nlist, const Gate& G, cudaStream_t st) {
  // API-level debug outputs (g, gL/gR, vstar mirrors; single rank): their own
  // instantiation, so the production kernel carries none of that code
  if (VISC && !elist && (D.g || D.gL || D.vstar))
    return elem2_kf<N, VISC, SHOCK, false, VISC>(D, P, U, elist, nlist, G, st);
  return elist ? elem2_kf<N, VISC, SHOCK, true, false>(D, P, U, elist, nlist, G, st)
               : elem2_kf<N, VISC, SHOCK, false, false>(D, P, U, elist, nlist, G, st);
}

template <int N>
static int elem_n(const hdg_domain& D, const hdg_params& P, const double* U, const int32_t* el,
                  int nl, const Gate& G, cudaStream_t st) {
  if constexpr (kElemPair<N>) {
    if (P.split && (!P.shock || P.viscous))
      return !P.viscous ? elem2_nf<N, false, false>(D, P, U, el, nl, G, st)
             : P.shock  ? elem2_nf<N, true, true>(D, P, U, el, nl, G, st)
                        : elem2_nf<N, true, false>(D, P, U, el, nl, G, st);
  }
  if (P.split)
    return P.viscous ? elem_nf<N, true, true>(D, P, U, el, nl, G, st)
                     : elem_nf<N, true, false>(D, P, U, el, nl, G, st);
  return P.viscous ? elem_nf<N, false, true>(D, P, U, el, nl, G, st)
                   : elem_nf<N, false, false>(D, P, U, el, nl, G, st);
}

// the FV kernel's producer claims elements from D.work[slot]; reset it on the stream
// (the element kernels keep a static round-robin: measured 1.7% faster on one GPU)
static int reset_work(const hdg_domain& D, int slot, cudaStream_t st) {
  if (!D.work) {
    hdg::set_error("hdg_domain.work (int32[4]) is required by the persistent kernels");
    return -1;
  }
  cudaError_t err = cudaMemsetAsync(D.work + slot, 0, sizeof(int32_t), st);
  if (err != cudaSuccess) {
    hdg::set_error("cudaMemsetAsync(work): %s", cudaGetErrorString(err));
    return -4;
  }
  return 0;
}

int run_elem(const hdg_domain& D, const hdg_params& P, const double* U, const int32_t* elist,
             int nlist, bool reset_fv, cudaStream_t st, const Gate* gate) {
  const Gate& G = gate ? *gate : kNoGate;
  if (P.shock && reset_fv) {
    if (!D.fv_count || !D.fv_list || !D.rfv) {
      hdg::set_error("shock capturing needs rfv / fv_list / fv_count workspaces");
      return -1;
    }
    // the element kernel appends flagged elements: reset the count on the stream
    cudaError_t err = cudaMemsetAsync(D.fv_count, 0, sizeof(int32_t), st);
    if (err != cudaSuccess) {
      hdg::set_error("cudaMemsetAsync(fv_count): %s", cudaGetErrorString(err));
      return -4;
    }
  }
#define CALL(n) elem_n<n>(D, P, U, elist, nlist, G, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

template <int N>
static int update_n(const hdg_domain& D, const hdg_params& P, const VolArgs& V,
                    const int32_t* elist, int nlist, const Gate& G, cudaStream_t st) {
  constexpr int n3 = (N + 1) * (N + 1) * (N + 1);
  const long total = (long)(elist ? nlist : D.ne) * n3;
  if (total <= 0) return 0;
  const int lserk = (V.mode & 15) != HDG_MODE_STORE_UT;
  if (lserk && ((V.mode >> 4) & 64)) {
    if (!D.dt_bits || !D.J) {
      hdg::set_error("the folded next-step dt needs dt_bits and J");
      return -1;
    }
    // 64-node blocks: measured 1-2 % faster than 128 / 256 at C2 and C4 (more, smaller
    // blocks in flight over the f* gather)
    update_kernel<N, true><<<(int)((total + 64 - 1) / 64), 64, 0, st>>>(D, P, V, elist, nlist, G);
  } else {
    update_kernel<N, false><<<(int)((total + 64 - 1) / 64), 64, 0, st>>>(D, P, V, elist, nlist, G);
  }
  return check_launch("update_kernel");
}

template <int N>
static int fv_n(const hdg_domain& D, const hdg_params& P, const double* U, cudaStream_t st) {
  using FD = FvDim<N>;
  static int blocks = -1;
  if (blocks < 0) {
    int rc = prep_kernel(fv_kernel<N>, FD::SMEM);
    if (rc) return rc;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fv_kernel<N>, FD::THREADS, FD::SMEM);
    blocks = sms * (per > 0 ? per : 1);
  }
  // persistent over the device-side flagged count (no host sync)
  if (int rc = reset_work(D, 1, st)) return rc;
  fv_kernel<N><<<blocks, FD::THREADS, FD::SMEM, st>>>(D, P, U);
  return check_launch("fv_kernel");
}

int run_update(const hdg_domain& D, const hdg_params& P, const VolArgs& V, const int32_t* elist,
               int nlist, bool do_fv, cudaStream_t st, const Gate* gate) {
  const Gate& G = gate ? *gate : kNoGate;
  if (P.shock && do_fv) {
    // FV residual of the elements the element kernel flagged, then the streaming update
    // blends it in after the Jacobian
    int rc;
#define CALLF(n) fv_n<n>(D, P, V.U, st)
    switch (D.N) {
      case 1: rc = CALLF(1); break;
      case 2: rc = CALLF(2); break;
      case 3: rc = CALLF(3); break;
      case 4: rc = CALLF(4); break;
      case 5: rc = CALLF(5); break;
      case 6: rc = CALLF(6); break;
      case 7: rc = CALLF(7); break;
      default: hdg::set_error("unsupported degree N=%d (1..7)", (int)D.N); return -2;
    }
#undef CALLF
    if (rc) return rc;
  }
#define CALL(n) update_n<n>(D, P, V, elist, nlist, G, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

template <int N>
static int peer_traces_n(const hdg_domain& D, const double* U, const int32_t* nbr,
                         const int32_t* src, const int32_t* dst, int n,
                         const unsigned long long* base, const unsigned long long* flags, int n_nbr,
                         unsigned* counter, unsigned long long* epoch, cudaStream_t st) {
  constexpr int n2 = (N + 1) * (N + 1);
  const long total = (long)n * n2;
  const long want = total > 0 ? (total + 255) / 256 : 1, cap = 2L * hdg::sm_count();
  const int blocks = (int)(want < cap ? want : cap);
  peer_send_traces_kernel<N><<<blocks, 256, 0, st>>>(D, U, nbr, src, dst, n, base, flags, n_nbr,
                                                      counter, epoch);
  return check_launch("peer_send_traces_kernel");
}

int run_peer_traces(const hdg_domain& D, const double* U, const int32_t* nbr, const int32_t* src,
                    const int32_t* dst, int n, const unsigned long long* base,
                    const unsigned long long* flags, int n_nbr, unsigned* counter,
                    unsigned long long* epoch, cudaStream_t st) {
#define CALL(nn) peer_traces_n<nn>(D, U, nbr, src, dst, n, base, flags, n_nbr, counter, epoch, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

template <int N>
static int pack_traces_n(const hdg_domain& D, const double* U, const int32_t* sides, int n,
                         double* buf, cudaStream_t st) {
  if (n <= 0) return 0;
  constexpr int n2 = (N + 1) * (N + 1);
  const long total = (long)n * n2;
  if (D.node_type == 0)
    pack_traces_kernel<N, true><<<(int)((total + 255) / 256), 256, 0, st>>>(D, U, sides, n, buf);
  else
    pack_traces_kernel<N, false><<<(int)((total + 255) / 256), 256, 0, st>>>(D, U, sides, n, buf);
  return check_launch("pack_traces_kernel");
}

int run_pack_traces(const hdg_domain& D, const double* U, const int32_t* sides, int n, double* buf,
                    cudaStream_t st) {
#define CALL(nn) pack_traces_n<nn>(D, U, sides, n, buf, st)
  HDG_DISPATCH_N(D.N, CALL)
#undef CALL
}

// E2_TIMING builds only: read and reset the element kernel's phase cycle counters
int read_phase_cycles(unsigned long long* out) {
#ifdef E2_TIMING
  cudaMemcpyFromSymbol(out, e2_cycles, sizeof(unsigned long long) * 8);
  const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(e2_cycles, z, sizeof(z));
  return 0;
#else
  for (int i = 0; i < 8; ++i) out[i] = 0;
  return -1;
#endif
}
