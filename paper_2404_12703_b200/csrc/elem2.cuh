// A for even n1 (N = 5, 7): the element pass of the Navier-Stokes / Euler split-form
// stage with two nodes per thread and a line-per-thread split-form volume integral.
// Included after elem.cuh in BOTH kernel sets: every phase evaluates the
// reference's operations in the reference's order, so the -fmad=false build is
// bit-identical to the reference and the FMA build is its contraction.
//
// Phases per element (one element per CTA, persistent over elements):
//   P1 prims + repack: thread t owns nodes (i,j,k) and (i,j,k+n1/2) -- both on the
//      same zeta line, so the zeta-partner reads of the lifting serve both nodes;
//   P2 vstar on the element's face nodes (k_lift_fill, src/operator.py:377-391);
//   P3 BR1 lifting (k_lift_volume :394-418, k_lift_surf_and_jac :421-453), the
//      contravariant viscous fluxes (k_viscous_contravariant :89-102) and the
//      element-side face viscous fluxes (k_fill_flux_viscous :295-330);
//   P4 the split-form volume integral exactly as k_vol_int_split (:142-209): one
//      thread per (direction, line), the unordered node pairs m <= al of the line,
//      each two-point flux F# (pt_split_flux_kep) evaluated ONCE and accumulated
//      into both nodes with Dsplit[m][al] / Dsplit[al][m] (Dsplit read from the
//      constant bank: all lanes use the same entry at the same time);
//   P5 Ut = ((0 + acc_xi) + acc_eta) + acc_zeta in the reference's direction order:
//      each line thread leaves its accumulators in its own nodes' direction slots of
//      MJ1 / WF (only it reads them), then every thread sums its two nodes' three
//      direction results and stores Vol.


// phase-time instrumentation (build with -DE2_TIMING only; tools/phase_times.py):
// thread 0 of every block adds the cycles between consecutive block-wide points
// (all phases end at a barrier) into e2_cycles[phase]
#ifdef E2_TIMING
__device__ unsigned long long e2_cycles[8];
#define E2_MARK(k)                                                   \
  do {                                                               \
    if (threadIdx.x == 0) {                                          \
      const long long now_ = clock64();                              \
      atomicAdd(&e2_cycles[k], (unsigned long long)(now_ - e2_t0));  \
      e2_t0 = now_;                                                  \
    }                                                                \
  } while (0)
#else
#define E2_MARK(k) do {} while (0)
#endif

template <int N>
__host__ __device__ constexpr int elem2_threads() {
  return ((Dim<N>::n3 / 2 + 31) / 32) * 32;
}

// shared-memory map (doubles) of elem2_kernel<N, VISC>
template <int N, bool VISC>
struct E2Map {
  using DM = Dim<N>;
  static constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3, PN = n2 * (n1 + 1);
  static constexpr int UB = (n3 * 5 + 3) & ~1, JB = (n3 * 9 + 3) & ~1;
  static constexpr int oSB = 0;
  static constexpr int oD4 = (DM::BASIS + 1) & ~1;           // [n2] 4 Dhat^T (lifting)
  static constexpr int oJ = oD4 + ((n2 + 1) & ~1);            // raw Ja block (TMA)
  static constexpr int oU = oJ + JB;                          // raw U block (TMA)
  static constexpr int oIJ = oU + UB;                         // 1/J block (TMA)
  static constexpr int oM1 = oIJ + DM::IJB;                   // [3][PN] Ja_z / 2
  static constexpr int oM2 = oM1 + 3 * PN;                    // [3][PN] (Ja_x, Ja_y) / 2
  static constexpr int oQ = oM2 + 6 * PN;                     // [4][PN] halved prim pairs
  static constexpr int oVS = oQ + 8 * PN;                     // [6][n2][4] face vstar
  static constexpr int oNV = oVS + (VISC ? 24 * n2 : 0);      // [6][NVB] nvec (TMA)
  static constexpr int oSS = oNV + (VISC ? 6 * DM::NVB : 0);  // [6][SSB] ssurf (TMA)
  static constexpr int oW = oSS + (VISC ? 6 * DM::SSB : 0);   // halved Fvis [3][2][PN] double2
  static constexpr int WORK = VISC ? 12 * PN : 0;
  // P4 accumulators: the viscous kernel reuses each direction's own MJ1 / WF slots;
  // the Euler kernel (no WF) has [3][5][PN] of its own
  static constexpr int oR = oW + WORK;
  static constexpr int RB = VISC ? 0 : 15 * PN;
  static constexpr int END = oR + RB;
  static constexpr size_t SMEM = sizeof(double) * END;
};

// stress tensor + heat flux of one node: t = (txx, tyy, tzz, txy, txz, tyz, qx, qy, qz),
// the operations of pt_viscous_flux_dir (src/equations.py:262-285) before the projection
__device__ __forceinline__ void stress_tensor(double mu, double lam, const double* g, double t[9]) {
  const double divu = g[0] + g[5] + g[10];
  t[0] = mu * (2.0 * g[0] - 2.0 / 3.0 * divu);
  t[1] = mu * (2.0 * g[5] - 2.0 / 3.0 * divu);
  t[2] = mu * (2.0 * g[10] - 2.0 / 3.0 * divu);
  t[3] = mu * (g[4] + g[1]);
  t[4] = mu * (g[8] + g[2]);
  t[5] = mu * (g[9] + g[6]);
  t[6] = -lam * g[3];
  t[7] = -lam * g[7];
  t[8] = -lam * g[11];
}

// the projection of pt_viscous_flux_dir from a prebuilt stress tensor (out[1..4])
__device__ __forceinline__ void stress_flux(const double t[9], double u, double v, double w,
                                            double nx, double ny, double nz, double out[5]) {
  out[1] = -(t[0] * nx + t[3] * ny + t[4] * nz);
  out[2] = -(t[3] * nx + t[1] * ny + t[5] * nz);
  out[3] = -(t[4] * nx + t[5] * ny + t[2] * nz);
  out[4] = (-(t[0] * u + t[3] * v + t[4] * w) + t[6]) * nx +
           (-(t[3] * u + t[1] * v + t[5] * w) + t[7]) * ny +
           (-(t[4] * u + t[5] * v + t[2] * w) + t[8]) * nz;
}

// ghost (replica) half of a Dirichlet side's viscous face flux: the BC state's
// prims with the element's gradient (gR = gL, src/operator.py:698-705)
__device__ __forceinline__ void face_viscous_bc(const hdg_domain& D, const Gas& G, int bc,
                                             const double* g, double nx, double ny, double nz,
                                             double* dr) {
  double ub[5], pb[7], fv[5];
  for (int v = 0; v < 5; ++v) ub[v] = D.bc_states[bc * 5 + v];
  prim_point(ub, pb, G);
  const double mub = viscosity(pb[5], G);
  const double lamb = conductivity(mub, G);
  viscous_flux_dir(pb[1], pb[2], pb[3], mub, lamb, g, nx, ny, nz, fv);
  for (int v = 1; v < 5; ++v) dr[v - 1] = fv[v];
}

// element-side viscous face fluxes of one node (k_fill_flux_viscous, :295-330, the
// element's half of the BR1 mean) on every face the node lies on: the projection of
// the node's stress tensor on the side's unit normal (pt_viscous_flux_dir)
template <int N, bool DBG>
__device__ __forceinline__ void face_viscous_tau(const hdg_domain& D, const Gas& G, int node,
                                                 const double tau[9], double u, double v,
                                                 double w, const double* g, const double* fnv,
                                                 const int* foff, const int* fef,
                                                 const int4* fsi) {
  constexpr int n1 = N + 1, n2 = n1 * n1;
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  // a node lies on at most one face per direction: one body per direction, in the
  // reference's ascending loc order
#pragma unroll
  for (int dir = 0; dir < 3; ++dir) {
    int m, a, b;
    face_coords(dir, i, j, k, m, a, b);
    if (m != 0 && m != N) continue;
    const int loc = 2 * dir + (m == N ? 1 : 0);
    const int info = fef[loc];
    const int s = info >> 3, rep = (info >> 2) & 1;
    int p, q;
    orient<N>(info & 3, a, b, p, q);
    const int fq = q * n1 + p;
    const double* nv = fnv + loc * Dim<N>::NVB + foff[2 * loc] + fq * 3;
    double fv[5];
    stress_flux(tau, u, v, w, nv[0], nv[1], nv[2], fv);
    double* dst = D.fvface + (((size_t)s * 2 + rep) * n2 + fq) * 4;
#pragma unroll
    for (int c = 1; c < 5; ++c) dst[c - 1] = fv[c];
    if (DBG && D.gL) {
      double* dg = (rep ? D.gR : D.gL) + ((size_t)s * n2 + fq) * 12;
      for (int c = 0; c < 12; ++c) dg[c] = g[c];
    }
    const int meta = fsi[loc].z;
    if (((meta >> 12) & 3) == HDG_SIDE_BC) {
      face_viscous_bc(D, G, (meta >> 8) & 15, g, nv[0], nv[1], nv[2],
                      D.fvface + (((size_t)s * 2 + 1) * n2 + fq) * 4);
      if (DBG && D.gL) {
        double* dg = D.gR + ((size_t)s * n2 + fq) * 12;
        for (int c = 0; c < 12; ++c) dg[c] = g[c];
      }
    }
  }
}

// BR1 lifting surface term + 1/J of one node (k_lift_surf_and_jac, :421-453, the
// reference's loc order; LGL: lhat vanishes off the face)
template <int N>
__device__ __forceinline__ void lift_surface_packed(const double* sb, const double* vs, int node,
                                                    double g[12], const double* fnv,
                                                    const double* fss, const int* foff,
                                                    const double* fij, const int* fef) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2;
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  // at most one face per direction (one body per direction, ascending loc order)
#pragma unroll
  for (int dir = 0; dir < 3; ++dir) {
    int m, a, b;
    face_coords(dir, i, j, k, m, a, b);
    if (m != 0 && m != N) continue;
    const int loc = 2 * dir + (m == N ? 1 : 0);
    const int info = fef[loc];
    const double sign = ((info >> 2) & 1) ? -1.0 : 1.0;
    const double lh = (m == N) ? sb[DM::oLhp + N] : sb[DM::oLhm];
    int p, q;
    orient<N>(info & 3, a, b, p, q);
    const int fq = q * n1 + p;
    const double* nvp = fnv + loc * DM::NVB + foff[2 * loc] + fq * 3;
    const double w = sign * lh * fss[loc * DM::SSB + foff[2 * loc + 1] + fq];
    const double* vsv = vs + (loc * n2 + a * n1 + b) * 4;
#pragma unroll
    for (int dd = 0; dd < 3; ++dd) {
      const double nd = w * nvp[dd];
#pragma unroll
      for (int l = 0; l < 4; ++l) g[dd * 4 + l] += nd * vsv[l];
    }
  }
  const double iw = fij[node];
#pragma unroll
  for (int c = 0; c < 12; ++c) g[c] *= iw;
}

// Hennemann modal indicator (k_indicator, src/shock.py:46-110) with two nodes per
// thread: rho*p in w[0:n3] (written by the repack), w[n3:3 n3] scratch. The modal
// transforms keep the reference's ascending-m sums; the three energy sums run in
// node order on one thread in the exact set and as a warp-shuffle tree in the fast
// set. Writes D.alpha[e] and appends a flagged element to D.fv_list.
template <int N>
__device__ void elem2_indicator(const hdg_domain& D, const hdg_params& P, const double* sb,
                                double* w, int e, bool act, int t) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3, H = n1 / 2, T = n3 / 2;
  __shared__ double s_red[3][32];   // fast set: warp-tree partials
  (void)s_red;
  double alpha = 0.0;
  if (P.indicator == 0) {
    const double* Vi = sb + DM::oVinv;
    const double* ind = w;
    double* t1 = w + n3;
    double* t2 = w + 2 * n3;
    const int i = t % n1, j = (t / n1) % n1, k0 = t / n2;
    if (act) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int k = k0 + r * H;
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < n1; ++m) acc += Vi[i * n1 + m] * ind[k * n2 + j * n1 + m];
        t1[t + r * T] = acc;
      }
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int k = k0 + r * H;
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < n1; ++m) acc += Vi[j * n1 + m] * t1[k * n2 + m * n1 + i];
        t2[t + r * T] = acc;
      }
    }
    __syncthreads();
    double a = 0.0, b = 0.0, c = 0.0;   // fast set: the energy partial sums
    (void)a;
    (void)b;
    (void)c;
    if (act) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int k = k0 + r * H;
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < n1; ++m) acc += Vi[k * n1 + m] * t2[m * n2 + j * n1 + i];
        if constexpr (kExact) {
          t1[t + r * T] = acc;   // modal coefficient, summed in node order below
        } else {
          const double m2 = acc * acc;
          a += m2;
          if (k < N && j < N && i < N) b += m2;
          if (k < N - 1 && j < N - 1 && i < N - 1) c += m2;
        }
      }
    }
    double total = 0.0, clip1 = 0.0, clip2 = 0.0;
    if constexpr (kExact) {
      __syncthreads();
      if (t == 0) {
        for (int nn = 0; nn < n3; ++nn) {
          const int ii = nn % n1, jj = (nn / n1) % n1, kk = nn / n2;
          const double v = t1[nn] * t1[nn];
          total += v;
          if (kk < N && jj < N && ii < N) clip1 += v;
          if (kk < N - 1 && jj < N - 1 && ii < N - 1) clip2 += v;
        }
      }
    } else {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, off);
        b += __shfl_xor_sync(0xffffffffu, b, off);
        c += __shfl_xor_sync(0xffffffffu, c, off);
      }
      if ((t & 31) == 0) {
        s_red[0][t >> 5] = a;
        s_red[1][t >> 5] = b;
        s_red[2][t >> 5] = c;
      }
      __syncthreads();
      if (t == 0) {
        for (int wi = 0; wi < (int)(blockDim.x >> 5); ++wi) {
          total += s_red[0][wi];
          clip1 += s_red[1][wi];
          clip2 += s_red[2][wi];
        }
      }
    }
    if (t == 0) {
      double energy = 0.0;
      if (total > 1e-300) energy = (total - clip1) / total;
      if (clip1 > 1e-300) {
        const double e2 = (clip1 - clip2) / clip1;
        if (e2 > energy) energy = e2;
      }
      double al = 1.0 / (1.0 + exp(P.ind_slope * (energy - P.ind_threshold)));
      if (al > P.alpha_max) al = P.alpha_max;
      if (al < P.alpha_min) al = 0.0;
      alpha = al;
    }
  } else {
    alpha = dmin(P.alpha_const, P.alpha_max);
  }
  if (t == 0) {
    D.alpha[e] = alpha;
    if (alpha > 0.0) D.fv_list[atomicAdd(D.fv_count, 1)] = e;
  }
}

template <int N, bool VISC, bool SHOCK, bool LISTED, bool DBG>
__global__ void __launch_bounds__(elem2_threads<N>(), 1)
    elem2_kernel(hdg_domain D, hdg_params P, const double* __restrict__ U,
                 const int32_t* __restrict__ elist, int nlist, Gate GT) {
  using DM = Dim<N>;
  using MP = E2Map<N, VISC>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3, H = n1 / 2, T = n3 / 2;
  constexpr int PN = MP::PN;
  constexpr int KOFF = H * n1 * (n1 + 1);     // padded offset of node + H*n2
  static_assert(n1 % 2 == 0 && DM::EPB == 1, "two nodes per thread need an even n1");
  static_assert(!SHOCK || VISC, "the indicator scratch lives in the viscous work area");
  static_assert(!VISC || MP::WORK >= 3 * n3 + 36 * n2, "staging room");
  static_assert(3 * n2 <= elem2_threads<N>(), "one thread per (direction, line)");
  extern __shared__ double smem[];
  __shared__ uint64_t bar[3];                 // raw Ja | U + 1/J | nvec + ssurf
  __shared__ int s_off[16];
  __shared__ int s_ef[2][6];
  __shared__ int4 s_si[2][6];
  double* sb = smem + MP::oSB;
  double* sD4 = smem + MP::oD4;
  double* sJ = smem + MP::oJ;
  double* sU = smem + MP::oU;
  double* sIJ = smem + MP::oIJ;
  double* MJ1 = smem + MP::oM1;
  double2* MJ2 = reinterpret_cast<double2*>(smem + MP::oM2);
  double2* Q = reinterpret_cast<double2*>(smem + MP::oQ);
  double* vs = smem + MP::oVS;
  double* sNV = smem + MP::oNV;
  double* sSS = smem + MP::oSS;
  double* w = smem + MP::oW;
  double2* WF = reinterpret_cast<double2*>(w);
  // P5 Vol rows [n3][5] (viscous): over the prim pairs Q, dead after P4; they leave by
  // one bulk TMA store issued by thread TSTORE (a thread of the last warp, which owns no
  // line in P4), whose read of Q is waited for before the next element's P1 writes Q
  double* vob = reinterpret_cast<double*>(Q);
  static_assert(!VISC || 8 * PN >= n3 * 5, "Vol rows over the prim pairs");
  constexpr int TSTORE = elem2_threads<N>() - 32;
  double* R = smem + MP::oR;

  // LISTED: an element list (multi-GPU passes; ids prefetched through a ring, the
  // optional in-kernel exchange gate); otherwise the contiguous element range
  constexpr bool listed = LISTED;
  const int ngroups = listed ? nlist : D.ne;
  const int t = threadIdx.x;
  // n3/2 node pairs, the rest idle (compile-time true when n3/2 is a warp multiple)
  const bool act = (T == elem2_threads<N>()) || t < T;
  const int i = t % n1, j = (t / n1) % n1, k0 = t / n2;
  const int pn0 = pnode<N>(t);
  const Gas G = make_gas(P);
  // P4 task of this thread: direction ld, line (c1, c2), padded node indices lp[m]
  const bool line_act = t < 3 * n2;
  const int ld = line_act ? t / n2 : 0, lc = t % n2, c1 = lc % n1, c2 = lc / n1;
  int lp[n1];
  {
    // xi: (k,j,i) = (c2,c1,m); eta: (c2,m,c1); zeta: (m,c2,c1) -- lane-fastest c1
    const int base = ld == 0 ? (c2 * n1 + c1) * (n1 + 1)
                             : (ld == 1 ? c2 * n1 * (n1 + 1) + c1 : c2 * (n1 + 1) + c1);
    const int stride = ld == 0 ? 1 : (ld == 1 ? n1 + 1 : n1 * (n1 + 1));
#pragma unroll
    for (int m = 0; m < n1; ++m) lp[m] = base + m * stride;
  }

  __shared__ int s_eid[3];
  auto issue_ja = [&](int e0) {
    const char* lj;
    unsigned bj;
    s_off[14] = aligned_span(D.Ja + (size_t)e0 * n3 * 9, (size_t)n3 * 9, lj, bj);
    tma_load_1d(sJ, lj, bj, &bar[0]);
    mbar_expect_tx(&bar[0], bj);
  };
  // U + 1/J (lanes 0, 1) and the 6 sides' nvec / ssurf (lanes 2..13) of element e0,
  // issued by the lanes of one warp in parallel; the byte totals reduced to lane 0
  // for the single expect-tx arrival of each barrier
  auto issue_u_warp = [&](int e0) {
    const int lane = t & 31;
    const char* lo = nullptr;
    unsigned by = 0;
    if (lane == 0) {
      s_off[15] = aligned_span(U + (size_t)e0 * n3 * 5, (size_t)n3 * 5, lo, by);
      tma_load_1d(sU, lo, by, &bar[1]);
    } else if (lane == 1) {
      s_off[13] = aligned_span(D.invJ + (size_t)e0 * n3, n3, lo, by);
      tma_load_1d(sIJ, lo, by, &bar[1]);
    }
    by += __shfl_xor_sync(0xffffffffu, by, 1);
    if (lane == 0) mbar_expect_tx(&bar[1], by);
  };
  auto issue_nv_warp = [&](int buf) {
    const int lane = t & 31;
    const char* lo = nullptr;
    unsigned by = 0;
    if (lane < 12) {
      const int loc = lane >> 1;
      const int sd = s_ef[buf][loc] >> 3;
      double* dst;
      if ((lane & 1) == 0) {
        s_off[2 * loc] = aligned_span(D.nvec + (size_t)sd * n2 * 3, n2 * 3, lo, by);
        dst = sNV + loc * DM::NVB;
      } else {
        s_off[2 * loc + 1] = aligned_span(D.ssurf + (size_t)sd * n2, n2, lo, by);
        dst = sSS + loc * DM::SSB;
      }
      tma_load_1d(dst, lo, by, &bar[2]);
    }
    unsigned total = by;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) total += __shfl_xor_sync(0xffffffffu, total, off);
    if (lane == 0) mbar_expect_tx(&bar[2], total);
  };
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  load_basis<N>(sb, D.basis);
  for (int x = t; x < n2; x += blockDim.x) {
    const int r = x / n1, c = x % n1;
    sD4[c * n1 + r] = 4.0 * D.basis[DM::oDhat + x];   // exact scaling of the halved operands
  }
  auto has_face = [&](int grp, int x) { return x < 6 && grp < ngroups; };
  if (LISTED && t == 0) {
    const int g0 = blockIdx.x, g1 = g0 + gridDim.x;
    s_eid[0] = g0 < ngroups ? elist[g0] : 0;
    s_eid[1] = g1 < ngroups ? elist[g1] : 0;
  }
  if (has_face(blockIdx.x, t)) {
    const int inf = D.ef_info[(size_t)(listed ? elist[blockIdx.x] : blockIdx.x) * 6 + t];
    s_ef[0][t] = inf;
    s_si[0][t] = reinterpret_cast<const int4*>(D.side_info)[inf >> 3];
  }
  __syncthreads();
  if (t < 32 && (int)blockIdx.x < ngroups) {
    const int e0 = LISTED ? s_eid[0] : (int)blockIdx.x;
    if (t == 0) issue_ja(e0);
    issue_u_warp(e0);
    if (VISC) issue_nv_warp(0);
  }
  // where face node f's neighbour trace lives (U, a halo row or a BC state), from the
  // face tables of buffer buf. Computed one element ahead by the threads that own no
  // line in P4 and kept in s_src (over vs: dead from the end of P3 to the next P2),
  // so the element top only issues the copies
  const double** s_src = reinterpret_cast<const double**>(vs);
  // only where the threads without a line fill whole warps (N = 7: warps 6, 7);
  // otherwise each thread resolves its sources at the element top
  constexpr bool kSrcAhead = (3 * n2) % 32 == 0 && elem2_threads<N>() - 3 * n2 >= 32;
  static_assert(!VISC || 24 * n2 >= 6 * n2, "s_src over vs");
  auto trace_src = [&](int f, int buf) {
    const int loc = f / n2, a = (f % n2) / n1, b = f % n1;
    const int info = s_ef[buf][loc];
    int p, q;
    orient<N>(info & 3, a, b, p, q);
    return trace_ptr<N>(D, U, s_si[buf][loc], info >> 3, 1 - ((info >> 2) & 1), q, p);
  };
  if (VISC && kSrcAhead) {
    for (int f = t; f < 6 * n2; f += elem2_threads<N>()) s_src[f] = trace_src(f, 0);
    __syncthreads();
  }

  int it = 0;
  bool gated = !LISTED || GT.n == 0;
#ifdef E2_TIMING
  long long e2_t0 = clock64();
#endif
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    const int nxt = grp + gridDim.x;
    const int cb = it & 1, nbuf = cb ^ 1;
    if (LISTED && !gated && grp >= GT.pos) {   // halo traces of the listed boundary elements
      gate_wait(GT);
      gated = true;
    }
    const int e = LISTED ? s_eid[it % 3] : grp;
    const int en = LISTED ? (nxt < ngroups ? s_eid[(it + 1) % 3] : 0) : nxt;
    if (LISTED && t == 0 && nxt + (int)gridDim.x < ngroups)
      cp_async4(&s_eid[(it + 2) % 3], elist + nxt + gridDim.x);   // visible after the last barrier
    const bool tab = has_face(nxt, t);
    if (tab) cp_async4(&s_ef[nbuf][t], D.ef_info + (size_t)en * 6 + t);
    // neighbours' face traces -> shared staging (face nodes t, t + T)
    int stg_off[2] = {0, 0};   // word offset of the trace in its staging slot
    if (VISC) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int f = t + r * T;
        if (act && f < 6 * n2) {
          const double* src = kSrcAhead ? s_src[f] : trace_src(f, cb);
          // the 40-byte trace in three async copies into a 6-double slot: 16+16+8
          // bytes when it starts 16-byte aligned, else 16+16+16 from 8 bytes before it
          // (the trace then starts at word 1 of the slot); never outside the trace's row
          const int odd = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
          stg_off[r] = odd;
          double* stg = w + 3 * n3 + f * 6;
          const double* s0 = src - odd;
          cp_async16(stg, s0);
          cp_async16(stg + 2, s0 + 2);
          if (odd) cp_async16(stg + 4, s0 + 4);
          else cp_async8(stg + 4, s0 + 4);
        }
      }
    }
    // ---- P1: prims, halved and packed -------------------------------------------
    mbar_wait(&bar[1], it & 1);
    mbar_wait(&bar[0], it & 1);
    E2_MARK(0);   // top of the element: neighbour staging issued, TMA blocks landed
    if (VISC) {   // the previous element's Vol rows have left Q
      if (t == TSTORE) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncthreads();
    }
    if (act) {
      const double* ub = sU + s_off[15];
      const double* ja = sJ + s_off[14];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int node = t + r * T, pn = pn0 + r * KOFF;
        double u[5], pr[7];
#pragma unroll
        for (int v = 0; v < 5; ++v) u[v] = ub[node * 5 + v];
        prim_point(u, pr, G);
        if (pr[0] <= 0.0 || pr[4] <= 0.0) atomicOr(&D.status[HDG_STATUS_BAD_PRIM], 1);
        if (SHOCK && P.indicator == 0) {
          // rho * p with the indicator's own pressure formula (src/shock.py:59-63)
          const double ppi = (G.gamma - 1.0) *
                             (u[4] - 0.5 * (u[1] * u[1] + u[2] * u[2] + u[3] * u[3]) / u[0]);
          w[node] = u[0] * ppi;
        }
        Q[pn] = make_double2(0.5 * pr[0], 0.5 * pr[1]);
        Q[PN + pn] = make_double2(0.5 * pr[2], 0.5 * pr[3]);
        Q[2 * PN + pn] = make_double2(0.5 * pr[4], 0.5 * pr[6]);
        Q[3 * PN + pn] = make_double2(0.5 * pr[5], u[4]);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double* jv = ja + (a * n3 + node) * 3;
          MJ2[a * PN + pn] = make_double2(0.5 * jv[0], 0.5 * jv[1]);
          MJ1[a * PN + pn] = 0.5 * jv[2];
        }
      }
    }
    if (tab) {
      cp_async_wait_all();
      cp_async16(&s_si[nbuf][t], reinterpret_cast<const int4*>(D.side_info) + (s_ef[nbuf][t] >> 3));
    }
    __syncthreads();
    E2_MARK(1);   // P1 prims + repack
    if (t == 0 && nxt < ngroups) issue_ja(en);   // raw Ja repacked: stream the next block
    if constexpr (SHOCK) elem2_indicator<N>(D, P, sb, w, e, act, t);
    if (VISC) {
      // ---- P2: vstar = mean of both traces' (u, v, w, T) on the face nodes ---------
      cp_async_wait_all();
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int f = t + r * T;
        if (act && f < 6 * n2) {
          const int loc = f / n2, a = (f % n2) / n1, b = f % n1;
          const double* stg = w + 3 * n3 + f * 6 + stg_off[r];
          double nb[5], pnb[7];
#pragma unroll
          for (int v = 0; v < 5; ++v) nb[v] = stg[v];
          prim_point(nb, pnb, G);
          const int on = pnode<N>(vol_node<N>(loc, a, b, (loc & 1) ? N : 0));
          const double2 q0 = Q[on], q1 = Q[PN + on];
          const double qT = Q[3 * PN + on].x;
          double* o = vs + f * 4;
          o[0] = 0.5 * (2.0 * q0.y + pnb[1]);
          o[1] = 0.5 * (2.0 * q1.x + pnb[2]);
          o[2] = 0.5 * (2.0 * q1.y + pnb[3]);
          o[3] = 0.5 * (2.0 * qT + pnb[5]);
          if (DBG && D.vstar) {   // API mirror: the side's owner writes (primary, or a BC replica)
            const int info = s_ef[cb][loc];
            if (!((info >> 2) & 1) || s_si[cb][loc].x < 0) {
              int p, q;
              orient<N>(info & 3, a, b, p, q);
              double* dv = D.vstar + ((size_t)(info >> 3) * n2 + q * n1 + p) * 4;
#pragma unroll
              for (int l = 0; l < 4; ++l) dv[l] = o[l];
            }
          }
        }
      }
      __syncthreads();
      E2_MARK(5);   // indicator + P2 vstar
      // ---- P3: lifting, viscous fluxes, face viscous fluxes -------------------------
      if (act) {
        const double* ij = sIJ + s_off[13];
        const int* fef = s_ef[cb];
        double g0[12], g1[12];
#pragma unroll
        for (int c = 0; c < 12; ++c) g0[c] = g1[c] = 0.0;
        // k_lift_volume (:394-418): per al, the three directions' terms summed, then
        // added; the zeta partner is shared by both nodes
#pragma unroll
        for (int al = 0; al < n1; ++al) {
          const double di = sD4[al * n1 + i], dj = sD4[al * n1 + j];
          const double dk0 = sD4[al * n1 + k0], dk1 = sD4[al * n1 + k0 + H];
          const int pk = pnode<N>(al * n2 + j * n1 + i);
          const double2 ak0 = Q[pk], ak1 = Q[PN + pk];
          const double akT = Q[3 * PN + pk].x;
          const double phi_k[4] = {ak0.y, ak1.x, ak1.y, akT};
          const double2 mk = MJ2[2 * PN + pk];
          const double ja2[3] = {mk.x, mk.y, MJ1[2 * PN + pk]};
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            double* g = r ? g1 : g0;
            const int k = k0 + r * H;
            const double dk = r ? dk1 : dk0;
            const int pi = pnode<N>(k * n2 + j * n1 + al), pj = pnode<N>(k * n2 + al * n1 + i);
            const double2 ai0 = Q[pi], ai1 = Q[PN + pi];
            const double aiT = Q[3 * PN + pi].x;
            const double2 aj0 = Q[pj], aj1 = Q[PN + pj];
            const double ajT = Q[3 * PN + pj].x;
            const double phi_i[4] = {ai0.y, ai1.x, ai1.y, aiT};
            const double phi_j[4] = {aj0.y, aj1.x, aj1.y, ajT};
            const double2 mi = MJ2[pi], mj = MJ2[PN + pj];
            const double ja0[3] = {mi.x, mi.y, MJ1[pi]};
            const double ja1[3] = {mj.x, mj.y, MJ1[PN + pj]};
#pragma unroll
            for (int dd = 0; dd < 3; ++dd) {
              const double jai = di * ja0[dd], jaj = dj * ja1[dd], jak = dk * ja2[dd];
#pragma unroll
              for (int l = 0; l < 4; ++l) {
                if constexpr (kExact) {
                  g[dd * 4 + l] += jai * phi_i[l] + jaj * phi_j[l] + jak * phi_k[l];
                } else {   // fast set: three chained FMAs into the accumulator
                  g[dd * 4 + l] = fma(jai, phi_i[l], g[dd * 4 + l]);
                  g[dd * 4 + l] = fma(jaj, phi_j[l], g[dd * 4 + l]);
                  g[dd * 4 + l] = fma(jak, phi_k[l], g[dd * 4 + l]);
                }
              }
            }
          }
        }
#ifdef E2_TIMING2   // finer P3 split (extra barriers; diagnostics only, N = 7)
        __syncthreads();
        E2_MARK(6);
#endif
        mbar_wait(&bar[2], it & 1);   // this element's nvec / ssurf blocks
        lift_surface_packed<N>(sb, vs, t, g0, sNV, sSS, s_off, ij, fef);
        lift_surface_packed<N>(sb, vs, t + T, g1, sNV, sSS, s_off, ij, fef);
#ifdef E2_TIMING2
        __syncthreads();
        E2_MARK(7);
#endif
        // contravariant viscous fluxes (halved metrics -> halved fluxes) and the
        // element-side face viscous fluxes
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const double* g = r ? g1 : g0;
          const int node = t + r * T, pn = pn0 + r * KOFF;
          if (DBG && D.g) {
            double* dg = D.g + ((size_t)e * n3 + node) * 12;
#pragma unroll
            for (int c = 0; c < 12; ++c) dg[c] = g[c];
          }
          const double2 q0 = Q[pn], q1 = Q[PN + pn];
          double pr[7];
          pr[1] = 2.0 * q0.y;
          pr[2] = 2.0 * q1.x;
          pr[3] = 2.0 * q1.y;
          const double mu = viscosity(2.0 * Q[3 * PN + pn].x, G);
          const double lam = conductivity(mu, G);
          double tau[9];
          stress_tensor(mu, lam, g, tau);
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            double fv[5];
            const double2 m2 = MJ2[a * PN + pn];
            stress_flux(tau, pr[1], pr[2], pr[3], m2.x, m2.y, MJ1[a * PN + pn], fv);
            WF[(a * 2 + 0) * PN + pn] = make_double2(fv[1], fv[2]);
            WF[(a * 2 + 1) * PN + pn] = make_double2(fv[3], fv[4]);
          }
          face_viscous_tau<N, DBG>(D, G, node, tau, pr[1], pr[2], pr[3], g, sNV, s_off, fef,
                                   s_si[cb]);
        }
      }
    }
    __syncthreads();   // Q / MJ / WF complete; U, 1/J, nvec, ssurf consumed
    E2_MARK(2);   // P3 lifting + viscous fluxes (Euler: indicator)
    if (t < 32 && nxt < ngroups) issue_u_warp(en);
    if (VISC && t >= TSTORE && nxt < ngroups) issue_nv_warp(nbuf);   // nvec / ssurf, next
    // ---- P4: split-form volume integral, one (direction, line) per thread ----------
    // Each line reads only its own nodes' direction-ld slots of MJ / WF, so its
    // accumulators go straight back into those slots (no barrier, no extra buffer)
    if (VISC && kSrcAhead && !line_act && nxt < ngroups) {   // next element's trace sources
      for (int f = t - 3 * n2; f < 6 * n2; f += elem2_threads<N>() - 3 * n2)
        s_src[f] = trace_src(f, nbuf);
    }
    if (line_act) {
      double acc[n1][5];
      // fast Navier-Stokes: two rows per sweep (bitwise the same sums; the exact set
      // and the Euler pass keep the one-row sweep, which fits their code in registers)
      if constexpr (kExact || !VISC) split_line<N, VISC>(Q, MJ2, MJ1, WF, ld, lp, acc);
      else split_line2<N, VISC>(Q, MJ2, MJ1, WF, ld, lp, acc);
#pragma unroll
      for (int m = 0; m < n1; ++m) {
        double* r0 = VISC ? reinterpret_cast<double*>(WF + (ld * 2 + 0) * PN + lp[m])
                          : R + (ld * 5 + 0) * PN + lp[m];
        if (VISC) {
          double* r1 = reinterpret_cast<double*>(WF + (ld * 2 + 1) * PN + lp[m]);
          r0[0] = acc[m][0];
          r0[1] = acc[m][1];
          r1[0] = acc[m][2];
          r1[1] = acc[m][3];
          MJ1[ld * PN + lp[m]] = acc[m][4];
        } else {
#pragma unroll
          for (int v = 0; v < 5; ++v) r0[v * PN] = acc[m][v];
        }
      }
    }
    __syncthreads();
    E2_MARK(3);   // P4 split-form volume integral
    // ---- P5: Ut = ((0 + acc_xi) + acc_eta) + acc_zeta (src/operator.py:201-209) ----
    if (act) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int node = t + r * T, pn = pn0 + r * KOFF;
        double ut[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double a[5];
          if (VISC) {
            const double2 w0 = WF[(d * 2 + 0) * PN + pn], w1 = WF[(d * 2 + 1) * PN + pn];
            a[0] = w0.x;
            a[1] = w0.y;
            a[2] = w1.x;
            a[3] = w1.y;
            a[4] = MJ1[d * PN + pn];
          } else {
#pragma unroll
            for (int v = 0; v < 5; ++v) a[v] = R[(d * 5 + v) * PN + pn];
          }
#pragma unroll
          for (int v = 0; v < 5; ++v) ut[v] += a[v];
        }
        // viscous: the element's Vol rows are assembled in shared memory (over Q) and
        // leave as ONE bulk TMA store; Euler: direct
        double* dst = VISC ? vob + node * 5 : D.vol + ((size_t)e * n3 + node) * 5;
#pragma unroll
        for (int v = 0; v < 5; ++v) dst[v] = ut[v];
      }
    }
    if (VISC) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // Vol rows -> TMA
    if (tab || (LISTED && t == 0)) cp_async_wait_all();
    __syncthreads();   // Q / MJ / w free for the next element
    E2_MARK(4);   // P5 direction sum + Vol store
    if (VISC && t == TSTORE) {
      asm volatile(
          "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
          "cp.async.bulk.commit_group;" ::"l"(D.vol + (size_t)e * n3 * 5),
          "r"(smem_u32(vob)), "r"((unsigned)(n3 * 5 * sizeof(double)))
          : "memory");
    }
  }
  if (VISC && t == TSTORE) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
