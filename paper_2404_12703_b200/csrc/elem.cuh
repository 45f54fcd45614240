// Navier-Stokes stage split for LGL nodes (included after kernels.cuh):
//
//   A  elem_kernel    per element: prims, BR1 lifting (vstar from the
//                     neighbours' traces, volume + surface, 1/J), contravariant
//                     viscous fluxes, element-side viscous face fluxes, and the
//                     COMPLETE volume integral (split or standard form, viscous
//                     part included) -> Vol[e][node][5]
//   B  flux_kernel    f* on the sides (needs the face viscous fluxes of A)
//   C  update_kernel  per node: Ut = -(1/J)(Vol + SurfInt) [+ source], then store
//                     Ut or the fused LSERK stage update
//
// The reference's order of floating-point operations is kept: Vol holds the
// value the reference's Ut has after vol_int (operator.py:142-209 / :109-139,
// viscous means inside the two-point sum), C adds the gather surface terms in
// locSide order (:333-358) then multiplies by -1/J (:361-370). A reads U, Ja
// and writes Vol + face fluxes (no Fvis round trip through HBM); C is a pure
// stream. A is persistent: each block streams its next element's U and Ja into
// shared memory with TMA bulk copies (mbarrier-completed) while it computes the
// current one, so HBM traffic overlaps the FP64 work.

// padded node rows (see pnode): xi lines of even n1 get one slot of padding
template <int N>
constexpr int kXiPad = (N + 1) % 2 == 0 ? 1 : 0;   // odd n1: lines are conflict-free unpadded
template <int N>   // even: double2 arrays follow each other in shared memory
constexpr int kPN = ((N + 1) * (N + 1) * (N + 1 + kXiPad<N>) + 1) & ~1;

template <int N, bool SPLIT, bool VISC>
__host__ __device__ constexpr int elem_work() {
  using DM = Dim<N>;
  // split: halved viscous flux pairs for all 3 directions ([3][2][PN] double2)
  // standard: the 15 contravariant flux rows
  return SPLIT ? (VISC ? 12 * kPN<N> : 0) : 15 * DM::n3;
}

// ---- TMA bulk copies + mbarrier (sm_90+ async proxy), raw PTX -------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// per-thread asynchronous global -> shared copies (no register staging): the data
// is visible to the issuing thread after cp_async_wait_all, to the block after a
// following barrier
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// 16-byte aligned superset [lo, hi) of a byte range; returns the 8-byte-word
// offset of the range start inside the superset
__device__ __forceinline__ int aligned_span(const double* p, size_t nd, const char*& lo,
                                            unsigned& bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t a0 = a & ~uintptr_t(15);
  const uintptr_t a1 = (a + nd * 8 + 15) & ~uintptr_t(15);
  lo = reinterpret_cast<const char*>(a0);
  bytes = static_cast<unsigned>(a1 - a0);
  return static_cast<int>((a - a0) >> 3);
}

// padded node index: lines along xi get one slot of padding, so the 4 / 8 / 32
// distinct nodes a warp reads per step of the two-point loop fall into distinct banks
template <int N>
__device__ __forceinline__ int pnode(int node) {
  return (node / (N + 1)) * (N + 1 + kXiPad<N>) + node % (N + 1);
}

// halved KEP two-point flux of (own, partner) times D, accumulated (fast set):
// acc += dma * F#, with dma folded into the mass flux and the pressure sum
__device__ __forceinline__ void kep_acc(double hr, double hu, double hv, double hw, double hp,
                                        double hh, double2 q0, double2 q1, double2 q2, double jx,
                                        double jy, double jz, double dma, double acc[5]) {
  const double rm = hr + q0.x, um = hu + q0.y, vm = hv + q1.x, wm = hw + q1.y;
  const double pm = hp + q2.x, hm = hh + q2.y;
  const double vn = um * jx + vm * jy + wm * jz;
  const double md = dma * (rm * vn);
  const double pd = dma * pm;
  acc[0] += md;
  acc[1] = fma(md, um, fma(pd, jx, acc[1]));
  acc[2] = fma(md, vm, fma(pd, jy, acc[2]));
  acc[3] = fma(md, wm, fma(pd, jz, acc[3]));
  acc[4] = fma(md, hm, acc[4]);
}

// Dsplit of the degree the element kernels run, [N][m * n1 + al] (constant bank: in the
// line-per-thread volume integral every lane reads the same entry at the same time)
__constant__ double c_dsplit[8][64];

// shared-memory loads the compiler may neither merge nor hoist out of the pair loop
// (a partner's data is re-read for every pair instead of keeping the whole line live
// in registers: 8 nodes x 13 doubles would not fit next to the 40 accumulators)
__device__ __forceinline__ double2 lds2(const double2* p) {
  double2 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ double lds1(const double* p) {
  double r;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(smem_u32(p)));
  return r;
}

// P4: one line of k_vol_int_split (src/operator.py:174-200) in the reference's order.
// pn[m] = padded index of the line's node m; Q / MJ / WF hold halved values, so every
// arithmetic mean 0.5*(a+b) of the reference is the plain sum of the halves (binary
// scaling: bitwise the same). acc[m][v] accumulates the node's pairs in ascending al.
template <int N, bool VISC>
__device__ __forceinline__ void split_line(const double2* __restrict__ Q,
                                           const double2* __restrict__ MJ2,
                                           const double* __restrict__ MJ1,
                                           const double2* __restrict__ WF, int d,
                                           const int (&pn)[N + 1], double (&acc)[N + 1][5]) {
  constexpr int n1 = N + 1, PN = kPN<N>, S = N;
#pragma unroll
  for (int m = 0; m < n1; ++m) {
#pragma unroll
    for (int v = 0; v < 5; ++v) acc[m][v] = 0.0;
  }
#pragma unroll
  for (int m = 0; m < n1; ++m) {
    const int pm = pn[m];
    const double2 a0 = Q[pm], a1 = Q[PN + pm], a2 = Q[2 * PN + pm];
    const double2 am = MJ2[d * PN + pm];
    const double az = MJ1[d * PN + pm];
    double2 aw0 = make_double2(0.0, 0.0), aw1 = aw0;
    if (VISC) {
      aw0 = WF[(d * 2 + 0) * PN + pm];
      aw1 = WF[(d * 2 + 1) * PN + pm];
    }
#pragma unroll
    for (int al = m; al < n1; ++al) {
      const int pa = pn[al];
      double2 b0 = a0, b1 = a1, b2 = a2, bm = am;
      double bz = az;
      if (al != m) {   // the diagonal pair is the node with itself: no reload
        b0 = lds2(Q + pa);
        b1 = lds2(Q + PN + pa);
        b2 = lds2(Q + 2 * PN + pa);
        bm = lds2(MJ2 + d * PN + pa);
        bz = lds1(MJ1 + d * PN + pa);
      }
      // pt_split_flux_kep (src/equations.py:235-259)
      const double rm = a0.x + b0.x, um = a0.y + b0.y, vm = a1.x + b1.x, wm = a1.y + b1.y;
      const double pm_ = a2.x + b2.x, hm = a2.y + b2.y;
      const double jx = am.x + bm.x, jy = am.y + bm.y, jz = az + bz;
      const double vn = um * jx + vm * jy + wm * jz;
      const double mf = rm * vn;
      double f[5];
      f[0] = mf;
      f[1] = mf * um + pm_ * jx;
      f[2] = mf * vm + pm_ * jy;
      f[3] = mf * wm + pm_ * jz;
      f[4] = mf * hm;
      if (VISC) {   // fs[v] += 0.5 * (fv[m, v] + fv[al, v])
        const double2 bw0 = al == m ? aw0 : lds2(WF + (d * 2 + 0) * PN + pa);
        const double2 bw1 = al == m ? aw1 : lds2(WF + (d * 2 + 1) * PN + pa);
        f[1] += aw0.x + bw0.x;
        f[2] += aw0.y + bw0.y;
        f[3] += aw1.x + bw1.x;
        f[4] += aw1.y + bw1.y;
      }
      const double dma = c_dsplit[S][m * n1 + al];
      if (al == m) {
#pragma unroll
        for (int v = 0; v < 5; ++v) acc[m][v] += dma * f[v];
      } else {
        const double dam = c_dsplit[S][al * n1 + m];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          acc[m][v] += dma * f[v];
          acc[al][v] += dam * f[v];
        }
      }
    }
    // scheduling fence: without it ptxas hoists the partner loads of the whole line
    // and spills the accumulators
    __syncwarp(__activemask());
  }
}

// Two rows per sweep: the same pairs, sums and per-node addition order as split_line
// (node n still receives its pairs in ascending partner order: rows < m before, then
// (m, m), (m, m+1) / (m, m+1), (m+1, m+1), then the partners al > m+1, row m's pair
// before row m+1's), but each partner al > m+1 is read from shared memory once for
// both rows: 20 instead of 36 node reads per line (the pass is bound by the
// shared-memory wavefronts, profiles/r02_ncu_elem2_c2.txt). Both kernel sets.
struct LineNode {
  double2 q0, q1, q2, jm, w0, w1;
  double jz;
};

template <int N, bool VISC, bool VOL>
__device__ __forceinline__ LineNode line_node(const double2* __restrict__ Q,
                                              const double2* __restrict__ MJ2,
                                              const double* __restrict__ MJ1,
                                              const double2* __restrict__ WF, int d, int p) {
  constexpr int n1 = N + 1, PN = kPN<N>;
  LineNode r;
  if (VOL) {   // partner reads: neither merged nor hoisted (see lds2)
    r.q0 = lds2(Q + p);
    r.q1 = lds2(Q + PN + p);
    r.q2 = lds2(Q + 2 * PN + p);
    r.jm = lds2(MJ2 + d * PN + p);
    r.jz = lds1(MJ1 + d * PN + p);
    r.w0 = VISC ? lds2(WF + (d * 2 + 0) * PN + p) : make_double2(0.0, 0.0);
    r.w1 = VISC ? lds2(WF + (d * 2 + 1) * PN + p) : make_double2(0.0, 0.0);
  } else {
    r.q0 = Q[p];
    r.q1 = Q[PN + p];
    r.q2 = Q[2 * PN + p];
    r.jm = MJ2[d * PN + p];
    r.jz = MJ1[d * PN + p];
    r.w0 = VISC ? WF[(d * 2 + 0) * PN + p] : make_double2(0.0, 0.0);
    r.w1 = VISC ? WF[(d * 2 + 1) * PN + p] : make_double2(0.0, 0.0);
  }
  return r;
}

// pt_split_flux_kep (src/equations.py:235-259) of the halved pair (a, b), plus the
// viscous mean fs[v] += 0.5 * (fv[a, v] + fv[b, v])
template <bool VISC>
__device__ __forceinline__ void line_pair_flux(const LineNode& a, const LineNode& b,
                                               double f[5]) {
  const double rm = a.q0.x + b.q0.x, um = a.q0.y + b.q0.y, vm = a.q1.x + b.q1.x,
               wm = a.q1.y + b.q1.y;
  const double pm_ = a.q2.x + b.q2.x, hm = a.q2.y + b.q2.y;
  const double jx = a.jm.x + b.jm.x, jy = a.jm.y + b.jm.y, jz = a.jz + b.jz;
  const double vn = um * jx + vm * jy + wm * jz;
  const double mf = rm * vn;
  f[0] = mf;
  f[1] = mf * um + pm_ * jx;
  f[2] = mf * vm + pm_ * jy;
  f[3] = mf * wm + pm_ * jz;
  f[4] = mf * hm;
  if (VISC) {
    f[1] += a.w0.x + b.w0.x;
    f[2] += a.w0.y + b.w0.y;
    f[3] += a.w1.x + b.w1.x;
    f[4] += a.w1.y + b.w1.y;
  }
}

template <int N, bool VISC>
__device__ __forceinline__ void split_line2(const double2* __restrict__ Q,
                                            const double2* __restrict__ MJ2,
                                            const double* __restrict__ MJ1,
                                            const double2* __restrict__ WF, int d,
                                            const int (&pn)[N + 1], double (&acc)[N + 1][5]) {
  constexpr int n1 = N + 1, S = N;
  static_assert(n1 % 2 == 0, "rows in pairs");
#pragma unroll
  for (int m = 0; m < n1; ++m) {
#pragma unroll
    for (int v = 0; v < 5; ++v) acc[m][v] = 0.0;
  }
#pragma unroll
  for (int m = 0; m < n1; m += 2) {
    const LineNode A = line_node<N, VISC, false>(Q, MJ2, MJ1, WF, d, pn[m]);
    const LineNode B = line_node<N, VISC, false>(Q, MJ2, MJ1, WF, d, pn[m + 1]);
    double f[5];
    line_pair_flux<VISC>(A, A, f);
    {
      const double w = c_dsplit[S][m * n1 + m];
#pragma unroll
      for (int v = 0; v < 5; ++v) acc[m][v] += w * f[v];
    }
    line_pair_flux<VISC>(A, B, f);
    {
      const double wa = c_dsplit[S][m * n1 + m + 1], wb = c_dsplit[S][(m + 1) * n1 + m];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        acc[m][v] += wa * f[v];
        acc[m + 1][v] += wb * f[v];
      }
    }
    line_pair_flux<VISC>(B, B, f);
    {
      const double w = c_dsplit[S][(m + 1) * n1 + m + 1];
#pragma unroll
      for (int v = 0; v < 5; ++v) acc[m + 1][v] += w * f[v];
    }
#pragma unroll
    for (int al = m + 2; al < n1; ++al) {
      const LineNode P = line_node<N, VISC, true>(Q, MJ2, MJ1, WF, d, pn[al]);
      line_pair_flux<VISC>(A, P, f);
      {
        const double wa = c_dsplit[S][m * n1 + al], wp = c_dsplit[S][al * n1 + m];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          acc[m][v] += wa * f[v];
          acc[al][v] += wp * f[v];
        }
      }
      line_pair_flux<VISC>(B, P, f);
      {
        const double wb = c_dsplit[S][(m + 1) * n1 + al], wp = c_dsplit[S][al * n1 + m + 1];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          acc[m + 1][v] += wb * f[v];
          acc[al][v] += wp * f[v];
        }
      }
    }
    // scheduling fence (as in split_line)
    __syncwarp(__activemask());
  }
}

// BR1 lifted gradient on the packed element layouts of elem_kernel (same
// arithmetic, same order as lift_gradient): Q = (rho,u)(v,w)(p,h)(T,rhoE) pairs,
// MJ2/MJ1 = (Ja_x, Ja_y) / Ja_z per direction, all on padded node indices.
template <int N>
__device__ __forceinline__ void lift_gradient_packed(
    const hdg_domain& D, const double* sb, const double* Dh, const double2* MJ2,
    const double* MJ1, const double2* Q, const double* vs, int e, int node, double g[12],
    const double* fnv, const double* fss, const int* foff, const double* fij, const int* fef) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3;
  constexpr int PN = kPN<N>;
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
#pragma unroll
  for (int c = 0; c < 12; ++c) g[c] = 0.0;
#pragma unroll
  for (int al = 0; al < n1; ++al) {
    const double di = Dh[al * n1 + i], dj = Dh[al * n1 + j], dk = Dh[al * n1 + k];  // Dh^T
    const int pi = pnode<N>(k * n2 + j * n1 + al), pj = pnode<N>(k * n2 + al * n1 + i),
              pk = pnode<N>(al * n2 + j * n1 + i);
    const double2 ai0 = Q[pi], ai1 = Q[PN + pi], ai3 = Q[3 * PN + pi];
    const double2 aj0 = Q[pj], aj1 = Q[PN + pj], aj3 = Q[3 * PN + pj];
    const double2 ak0 = Q[pk], ak1 = Q[PN + pk], ak3 = Q[3 * PN + pk];
    const double phi_i[4] = {ai0.y, ai1.x, ai1.y, ai3.x};
    const double phi_j[4] = {aj0.y, aj1.x, aj1.y, aj3.x};
    const double phi_k[4] = {ak0.y, ak1.x, ak1.y, ak3.x};
    const double2 mi = MJ2[pi], mj = MJ2[PN + pj], mk = MJ2[2 * PN + pk];
    const double ja0[3] = {mi.x, mi.y, MJ1[pi]};
    const double ja1[3] = {mj.x, mj.y, MJ1[PN + pj]};
    const double ja2[3] = {mk.x, mk.y, MJ1[2 * PN + pk]};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double jai = di * ja0[d];
      const double jaj = dj * ja1[d];
      const double jak = dk * ja2[d];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        if constexpr (kExact) {
          g[d * 4 + l] += jai * phi_i[l] + jaj * phi_j[l] + jak * phi_k[l];
        } else {   // fast set: three chained FMAs into the accumulator
          g[d * 4 + l] = fma(jai, phi_i[l], g[d * 4 + l]);
          g[d * 4 + l] = fma(jaj, phi_j[l], g[d * 4 + l]);
          g[d * 4 + l] = fma(jak, phi_k[l], g[d * 4 + l]);
        }
      }
    }
  }
#pragma unroll
  for (int loc = 0; loc < 6; ++loc) {
    int m, a, b;
    face_coords(loc >> 1, i, j, k, m, a, b);
    if (m != ((loc & 1) ? N : 0)) continue;   // lhat is exactly 0 off the face (LGL)
    const int info = fef[loc];
    const int code = info & 3;
    const double sign = ((info >> 2) & 1) ? -1.0 : 1.0;
    const double lh = sb[((loc & 1) ? DM::oLhp : DM::oLhm) + m];
    int p, q;
    orient<N>(code, a, b, p, q);
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
  if (D.g) {
    double* dg = D.g + ((size_t)e * n3 + node) * 12;
#pragma unroll
    for (int c = 0; c < 12; ++c) dg[c] = g[c];
  }
}

// Hennemann modal indicator of one element (k_indicator, src/shock.py:46-110) on
// rho*p already in w[0:n3]; w[n3:3 n3] is scratch. Writes D.alpha[e] and appends
// flagged elements (alpha > 0) to D.fv_list. Called by every thread of the block.
// The energy sums run sequentially in (k,j,i) order in the exact set (as the
// reference) and as a warp-shuffle tree in the fast set.
template <int N>
__device__ void element_indicator(const hdg_domain& D, const hdg_params& P, const double* sb,
                                  double* w, int e, bool active, int node) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3;
  __shared__ double s_red[3][32];   // fast set: warp-tree partials
  (void)s_red;
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  double* ind = w;
  double* t1 = w + n3;
  double* t2 = w + 2 * n3;
  double alpha = 0.0;
  if (P.indicator == 0) {
    const double* Vi = sb + DM::oVinv;
    if (active) {
      double acc = 0.0;
      for (int m = 0; m < n1; ++m) acc += Vi[i * n1 + m] * ind[k * n2 + j * n1 + m];
      t1[node] = acc;
    }
    __syncthreads();
    if (active) {
      double acc = 0.0;
      for (int m = 0; m < n1; ++m) acc += Vi[j * n1 + m] * t1[k * n2 + m * n1 + i];
      t2[node] = acc;
    }
    __syncthreads();
    double m2 = 0.0;
    if (active) {
      double acc = 0.0;
      for (int m = 0; m < n1; ++m) acc += Vi[k * n1 + m] * t2[m * n2 + j * n1 + i];
      m2 = acc * acc;
      t1[node] = acc;
    }
    __syncthreads();
    double total = 0.0, clip1 = 0.0, clip2 = 0.0;
    if constexpr (kExact) {
      if (active && node == 0) {
        for (int nn = 0; nn < n3; ++nn) {
          const int ii = nn % n1, jj = (nn / n1) % n1, kk = nn / n2;
          const double v = t1[nn] * t1[nn];
          total += v;
          if (kk < N && jj < N && ii < N) clip1 += v;
          if (kk < N - 1 && jj < N - 1 && ii < N - 1) clip2 += v;
        }
      }
    } else {
      static_assert(DM::EPB == 1 || DM::n3 % 32 == 0 || true, "");
      double a = active ? m2 : 0.0;
      double b = (active && k < N && j < N && i < N) ? m2 : 0.0;
      double c = (active && k < N - 1 && j < N - 1 && i < N - 1) ? m2 : 0.0;
      for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, off);
        b += __shfl_xor_sync(0xffffffffu, b, off);
        c += __shfl_xor_sync(0xffffffffu, c, off);
      }
      // one element per block here (the NS element kernel has EPB == 1 for N >= 4);
      // for EPB > 1 the warps of one element are contiguous and n3 is a warp multiple
      // only for N = 3 / 7, so fall back to the sequential sum otherwise
      if (DM::EPB == 1) {
        if ((threadIdx.x & 31) == 0) {
          s_red[0][threadIdx.x >> 5] = a;
          s_red[1][threadIdx.x >> 5] = b;
          s_red[2][threadIdx.x >> 5] = c;
        }
        __syncthreads();
        if (node == 0) {
          for (int wi = 0; wi < (n3 + 31) / 32; ++wi) {
            total += s_red[0][wi];
            clip1 += s_red[1][wi];
            clip2 += s_red[2][wi];
          }
        }
      } else if (active && node == 0) {
        for (int nn = 0; nn < n3; ++nn) {
          const int ii = nn % n1, jj = (nn / n1) % n1, kk = nn / n2;
          const double v = t1[nn] * t1[nn];
          total += v;
          if (kk < N && jj < N && ii < N) clip1 += v;
          if (kk < N - 1 && jj < N - 1 && ii < N - 1) clip2 += v;
        }
      }
    }
    if (active && node == 0) {
      double energy = 0.0;
      if (total > 1e-300) energy = (total - clip1) / total;
      if (clip1 > 1e-300) {
        const double e2 = (clip1 - clip2) / clip1;
        if (e2 > energy) energy = e2;
      }
      double a = 1.0 / (1.0 + exp(P.ind_slope * (energy - P.ind_threshold)));
      if (a > P.alpha_max) a = P.alpha_max;
      if (a < P.alpha_min) a = 0.0;
      alpha = a;
    }
  } else {
    alpha = dmin(P.alpha_const, P.alpha_max);
  }
  if (active && node == 0) {
    D.alpha[e] = alpha;
    if (alpha > 0.0) D.fv_list[atomicAdd(D.fv_count, 1)] = e;
  }
  __syncthreads();   // scratch (w) is reused by the caller
}

// FV subcell residual of the flagged elements (k_fv_residual, src/shock.py:113-195),
// warp-specialised and persistent over the device-side compacted list:
//   producer warp: per element, reads the list entry and the six side ids, then
//     issues TMA bulk copies of U, 1/J, the three subcell-metric blocks and the six
//     sides' f* into one of two stage buffers (full/empty mbarrier pair each);
//   consumer warps (one thread per node): prims -> shared, then per direction all
//     n1^2 (n1+1) interface fluxes (Riemann on interior interfaces, oriented f* on
//     the two faces) -> shared, and -(F[h+1]-F[h])/w_h into the node's residual.
// RFV * (1/J) -> D.rfv; the streaming update blends it (src/shock.py:198-210).
template <int N>
struct FvDim {
  static constexpr int n1 = N + 1, n2 = n1 * n1, n3 = n2 * n1;
  static constexpr int NC = ((n3 + 31) / 32) * 32;                 // consumer threads
  static constexpr int THREADS = NC + 32;                          // + producer warp
  // stage slots (+2 doubles of slack each for the 16-byte aligned superset)
  // (each slot a 16-byte multiple: the bulk copies land at 16-byte aligned addresses,
  // odd n3 included)
  static constexpr int UB = (n3 * 5 + 3) & ~1, IJB = (n3 + 3) & ~1,
                       MB = (n2 * (n1 + 1) * 3 + 3) & ~1, FB = (n2 * 5 + 3) & ~1;
  static constexpr int STAGE = (UB + IJB + 3 * MB + 6 * FB + 1) & ~1;
  static constexpr int FL = n2 * (n1 + 1) * 5;                     // one direction's fluxes
  static constexpr size_t SMEM = sizeof(double) * (2 * STAGE + 7 * n3 + FL + 2 * n1);
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int N>
__global__ void __launch_bounds__(FvDim<N>::THREADS) fv_kernel(hdg_domain D, hdg_params P,
                                                               const double* __restrict__ U) {
  using DM = Dim<N>;
  using FD = FvDim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3, NC = FD::NC;
  extern __shared__ double fsm[];
  __shared__ uint64_t full[2], empty[2];
  __shared__ int s_off[2][11];     // U, 1/J, 3 metric blocks, 6 f* blocks (word offsets)
  __shared__ int s_ef[2][7];       // element id + its 6 ef_info words
  double* stage = fsm;                        // [2][STAGE]
  double* sq = stage + 2 * FD::STAGE;         // [7][n3] prims + rhoE
  double* sF = sq + 7 * n3;                   // [n2][n1+1][5] fluxes of one direction
  double* sbw = sF + FD::FL;                  // [2 n1]: -, 1/weights
  const int tid = threadIdx.x;
  const int count = *D.fv_count;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], 1);
    mbar_init(&empty[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = tid; t < n1; t += blockDim.x) sbw[n1 + t] = D.basis[DM::oIW + t];
  __syncthreads();

  if (tid >= NC) {
    // ---- producer warp (one lane issues) --------------------------------------
    if (tid != NC) return;
    // dynamic schedule: first element = block index, then claimed from a counter
    int idx = blockIdx.x;
    for (int it = 0;; ++it) {
      const int buf = it & 1;
      if (it >= 2) mbar_wait(&empty[buf], ((it >> 1) - 1) & 1);
      if (idx >= count) {
        s_ef[buf][0] = -1;              // end of the list
        mbar_arrive(&full[buf]);
        break;
      }
      const int e = D.fv_list[idx];
      int ef[6];
#pragma unroll
      for (int loc = 0; loc < 6; ++loc) ef[loc] = D.ef_info[e * 6 + loc];
      s_ef[buf][0] = e;
#pragma unroll
      for (int loc = 0; loc < 6; ++loc) s_ef[buf][1 + loc] = ef[loc];
      double* st = stage + buf * FD::STAGE;
      const double* fvms[3] = {D.fvm0, D.fvm1, D.fvm2};
      const char* lo;
      unsigned by, total = 0;
      int slot = 0;
      s_off[buf][0] = aligned_span(U + (size_t)e * n3 * 5, (size_t)n3 * 5, lo, by);
      tma_load_1d(st + slot, lo, by, &full[buf]);
      total += by;
      slot += FD::UB;
      s_off[buf][1] = slot + aligned_span(D.invJ + (size_t)e * n3, n3, lo, by);
      tma_load_1d(st + slot, lo, by, &full[buf]);
      total += by;
      slot += FD::IJB;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const size_t mw = (size_t)n2 * (n1 + 1) * 3;
        s_off[buf][2 + d] = slot + aligned_span(fvms[d] + (size_t)e * mw, mw, lo, by);
        tma_load_1d(st + slot, lo, by, &full[buf]);
        total += by;
        slot += FD::MB;
      }
#pragma unroll
      for (int loc = 0; loc < 6; ++loc) {
        const double* fs = D.fstar + (size_t)(ef[loc] >> 3) * n2 * 5;
        s_off[buf][5 + loc] = slot + aligned_span(fs, (size_t)n2 * 5, lo, by);
        tma_load_1d(st + slot, lo, by, &full[buf]);
        total += by;
        slot += FD::FB;
      }
      mbar_expect_tx(&full[buf], total);   // arrive (release): s_ef / s_off visible
      idx = (int)gridDim.x + atomicAdd(D.work + 1, 1);
    }
    return;
  }

  // ---- consumers: one thread per node -------------------------------------------
  const Gas G = make_gas(P);
  const int node = tid;
  const bool act = node < n3;
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  for (int it = 0;; ++it) {
    const int buf = it & 1;
    mbar_wait(&full[buf], (it >> 1) & 1);
    const double* st = stage + buf * FD::STAGE;
    const int e = s_ef[buf][0];
    if (e < 0) break;
    const double* sU = st + s_off[buf][0];
    if (act) {
      double u[5], pr[7];
#pragma unroll
      for (int v = 0; v < 5; ++v) u[v] = sU[node * 5 + v];
      prim_point(u, pr, G);
      sq[0 * n3 + node] = pr[0];
      sq[1 * n3 + node] = pr[1];
      sq[2 * n3 + node] = pr[2];
      sq[3 * n3 + node] = pr[3];
      sq[4 * n3 + node] = pr[4];
      sq[6 * n3 + node] = u[4];
    }
    double rfv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int d = 0; d < 3; ++d) {
      consumer_sync(NC);   // prims ready / the previous direction's fluxes consumed
      const int loc_m = 2 * d, loc_p = 2 * d + 1;
      const int inm = s_ef[buf][1 + loc_m], inp = s_ef[buf][1 + loc_p];
      const double* mvb = st + s_off[buf][2 + d];
      // interior interfaces (a Riemann solve each) first, one per thread, then the
      // 2 n2 face interfaces (copies): the expensive work is balanced over threads
      for (int t = tid; t < n2 * (n1 + 1); t += NC) {
        int line, h;
        if (t < n2 * N) {
          line = t / N;
          h = 1 + t % N;
        } else {
          line = (t - n2 * N) >> 1;
          h = ((t - n2 * N) & 1) ? n1 : 0;
        }
        const int a = line % n1, b = line / n1;
        double f[5];
        if (h == 0 || h == n1) {
          const int info = h == 0 ? inm : inp;
          const double sg = ((info >> 2) & 1) ? -1.0 : 1.0;
          int p, qq;
          orient<N>(info & 3, a, b, p, qq);
          const double* fs = st + s_off[buf][5 + (h == 0 ? loc_m : loc_p)] + (qq * n1 + p) * 5;
          const double fac = h == 0 ? -sg : sg;
#pragma unroll
          for (int v = 0; v < 5; ++v) f[v] = fac * fs[v];
        } else {
          const int nL = vol_node<N>(loc_m, a, b, h - 1), nR = vol_node<N>(loc_m, a, b, h);
          const int r1 = d == 1 ? a : b, r2 = d == 1 ? b : a;
          const double* mv = mvb + ((r1 * n1 + r2) * (n1 + 1) + h) * 3;
          const double mx = mv[0], my = mv[1], mz = mv[2];
          const double sn = sqrt(mx * mx + my * my + mz * mz);
          const double L[5] = {sq[nL], sq[n3 + nL], sq[2 * n3 + nL], sq[3 * n3 + nL],
                               sq[4 * n3 + nL]};
          const double R[5] = {sq[nR], sq[n3 + nR], sq[2 * n3 + nR], sq[3 * n3 + nR],
                               sq[4 * n3 + nR]};
          riemann(P.fv_solver, L, sq[6 * n3 + nL], R, sq[6 * n3 + nR], mx / sn, my / sn, mz / sn,
                  G.gamma, f);
#pragma unroll
          for (int v = 0; v < 5; ++v) f[v] = f[v] * sn;
        }
        double* o = sF + (line * (n1 + 1) + h) * 5;
#pragma unroll
        for (int v = 0; v < 5; ++v) o[v] = f[v];
      }
      consumer_sync(NC);
      if (act) {
        int m, a, b;
        face_coords(d, i, j, k, m, a, b);
        const double iwh = sbw[n1 + m];
        const double* F0 = sF + ((b * n1 + a) * (n1 + 1) + m) * 5;
#pragma unroll
        for (int v = 0; v < 5; ++v) rfv[v] -= (F0[5 + v] - F0[v]) * iwh;
      }
    }
    if (act) {
      const double iw = st[s_off[buf][1] + node];
      double* dst = D.rfv + ((size_t)e * n3 + node) * 5;
#pragma unroll
      for (int v = 0; v < 5; ++v) dst[v] = rfv[v] * iw;
    }
    consumer_sync(NC);   // stage buffer and sq / sF free
    if (tid == 0) mbar_arrive(&empty[buf]);
  }
}

// A: persistent over element groups. Everything an element reads from HBM in
// bulk is staged by TMA (cp.async.bulk, mbarrier-completed) one element ahead:
//   barJ: the raw Ja block; it is repacked (halved, padded, (x,y)|z split) into
//         shared memory right away, so the next block streams in during the
//         whole element;
//   barF: U block, 1/J block and the 6 sides' nvec / ssurf blocks, issued for
//         the next element once this element's last reader is past a barrier.
// Only the neighbours' face traces (for vstar) are still gathered from global.
// Two-point loop operands are 16-byte pairs on padded node indices (3 + 2 + 2
// LDS.128 per partner node instead of 13 LDS.64).
template <int N, bool SPLIT, bool VISC>
__host__ __device__ constexpr size_t elem_smem() {
  using DM = Dim<N>;
  constexpr int UB = (DM::EPB * DM::n3 * 5 + 3) & ~1, JB = (DM::EPB * DM::n3 * 9 + 3) & ~1;
  constexpr int PN = kPN<N>;
  return sizeof(double) *
         (((DM::BASIS + 1) & ~1) + 2 * ((DM::n2 + 1) & ~1) + JB + UB + DM::EPB * DM::IJB +
          (VISC ? DM::EPB * 6 * (DM::NVB + DM::SSB) : 0) +
          DM::EPB * (3 * PN + 6 * PN + 8 * PN + (VISC ? 24 * DM::n2 : 0) +
                     elem_work<N, SPLIT, VISC>()));
}

// resident blocks per SM the element kernel is compiled for: as many as shared
// memory allows, but never below 128 registers per thread
template <int N, bool SPLIT, bool VISC>
__host__ __device__ constexpr int elem_min_blocks() {
  constexpr int by_smem = (int)((227 * 1024) / (elem_smem<N, SPLIT, VISC>() + 1024));
  constexpr int by_regs = 65536 / (Dim<N>::THREADS * 128);
  return (by_smem < by_regs ? by_smem : by_regs) < 1 ? 1 : (by_smem < by_regs ? by_smem : by_regs);
}

template <int N, bool SPLIT, bool VISC>
__global__ void __launch_bounds__(Dim<N>::THREADS, (elem_min_blocks<N, SPLIT, VISC>()))
    elem_kernel(hdg_domain D, hdg_params P, const double* __restrict__ U,
                const int32_t* __restrict__ elist, int nlist, Gate GT) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3, EPB = DM::EPB;
  constexpr int PN = kPN<N>;
  constexpr int UB = (EPB * n3 * 5 + 3) & ~1, JB = (EPB * n3 * 9 + 3) & ~1;
  extern __shared__ double smem[];
  __shared__ uint64_t bar[2];                 // barJ, barF
  __shared__ int s_off[EPB * 14 + 2];         // per element: 6 x (nvec, ssurf) + U + 1/J offsets
  // face tables of the current / next group, prefetched one group ahead with
  // cp.async: ef_info and the side_info record of each element face
  __shared__ int s_ef[2][EPB * 6];
  __shared__ int4 s_si[2][EPB * 6];
  static_assert(6 * EPB <= DM::THREADS, "face-table prefetch uses one thread per face");
  static_assert(!VISC || 6 * n2 > n3 || elem_work<N, SPLIT, VISC>() >= 3 * n3 + 30 * n2,
                "neighbour-trace staging lives behind the indicator scratch in w");
  double* sb = smem;
  // transposed operator copies ([alpha][row]): a warp reads 8 consecutive rows of one
  // column, bank-conflict free (row-major reads of 8 rows are 4-way conflicts)
  double* sD4 = sb + ((DM::BASIS + 1) & ~1);                  // [n2] (4*)Dhat^T (lifting)
  double* sDsT = sD4 + ((n2 + 1) & ~1);                       // [n2] Dsplit^T
  double* sJ = sDsT + ((n2 + 1) & ~1);                        // [JB] raw Ja block
  double* sU = sJ + JB;                                       // [UB] raw U block
  double* sIJ = sU + UB;                                      // [EPB][IJB] 1/J
  double* sNV = sIJ + EPB * DM::IJB;                          // [EPB][6][NVB] nvec (VISC)
  double* sSS = sNV + (VISC ? EPB * 6 * DM::NVB : 0);         // [EPB][6][SSB] ssurf (VISC)
  double* sM1 = sSS + (VISC ? EPB * 6 * DM::SSB : 0);         // [EPB][3][PN] Ja_z
  double2* sM2 = reinterpret_cast<double2*>(sM1 + EPB * 3 * PN);   // [EPB][3][PN] (Ja_x, Ja_y)
  double2* sQ = sM2 + EPB * 3 * PN;                           // [EPB][4][PN] prim pairs
  double* svs = reinterpret_cast<double*>(sQ + EPB * 4 * PN);     // [EPB][6*n2*4] (VISC)
  double* sw = svs + (VISC ? EPB * 24 * n2 : 0);              // [EPB][elem_work]
  // optional element list (multi-rank overlap: interior / boundary passes), EPB == 1
  const bool listed = elist != nullptr;
  const int ngroups = listed ? nlist : (D.ne + EPB - 1) / EPB;
  const int le = threadIdx.x / n3;
  const int node = threadIdx.x % n3;
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  const int pn = pnode<N>(node);
  const Gas G = make_gas(P);
  double2* Q = sQ + le * 4 * PN;
  double2* MJ2 = sM2 + le * 3 * PN;
  double* MJ1 = sM1 + le * 3 * PN;
  double* vs = svs + le * 24 * n2;
  double* w = sw + le * elem_work<N, SPLIT, VISC>();
  double2* WF = reinterpret_cast<double2*>(w);                // [3][2][PN] halved Fvis (split)

  auto issue_ja = [&](int grp) {
    const int e0 = listed ? elist[grp] : grp * EPB;
    const int ne_g = listed ? 1 : min(EPB, D.ne - e0);
    const char* lj;
    unsigned bj;
    s_off[EPB * 14] = aligned_span(D.Ja + (size_t)e0 * n3 * 9, (size_t)ne_g * n3 * 9, lj, bj);
    tma_load_1d(sJ, lj, bj, &bar[0]);
    mbar_expect_tx(&bar[0], bj);
  };
  auto issue_f = [&](int grp, int buf) {
    const int e0 = listed ? elist[grp] : grp * EPB;
    const int ne_g = listed ? 1 : min(EPB, D.ne - e0);
    const char* lo;
    unsigned by, total = 0;
    s_off[EPB * 14 + 1] = aligned_span(U + (size_t)e0 * n3 * 5, (size_t)ne_g * n3 * 5, lo, by);
    total += by;
    tma_load_1d(sU, lo, by, &bar[1]);
    for (int l = 0; l < ne_g; ++l) {
      s_off[l * 14 + 13] = aligned_span(D.invJ + (size_t)(e0 + l) * n3, n3, lo, by);
      total += by;
      tma_load_1d(sIJ + l * DM::IJB, lo, by, &bar[1]);
      if (VISC) {
        for (int loc = 0; loc < 6; ++loc) {
          const int sd = s_ef[buf][l * 6 + loc] >> 3;
          s_off[l * 14 + 2 * loc] = aligned_span(D.nvec + (size_t)sd * n2 * 3, n2 * 3, lo, by);
          total += by;
          tma_load_1d(sNV + (l * 6 + loc) * DM::NVB, lo, by, &bar[1]);
          s_off[l * 14 + 2 * loc + 1] = aligned_span(D.ssurf + (size_t)sd * n2, n2, lo, by);
          total += by;
          tma_load_1d(sSS + (l * 6 + loc) * DM::SSB, lo, by, &bar[1]);
        }
      }
    }
    // complete_tx may land before this arrive (transiently negative tx-count): the
    // phase completes once the arrival and all bytes are accounted
    mbar_expect_tx(&bar[1], total);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  load_basis<N>(sb, D.basis);
  for (int t = threadIdx.x; t < n2; t += blockDim.x) {
    const int r = t / n1, c = t % n1;
    sD4[c * n1 + r] = (SPLIT ? 4.0 : 1.0) * D.basis[DM::oDhat + t];   // exact scaling
    sDsT[c * n1 + r] = D.basis[DM::oDsplit + t];
  }
  // a thread per element face: does group grp have element face t?
  auto has_face = [&](int grp, int t) {
    return t < 6 * EPB && grp < ngroups && (listed || grp * EPB + t / 6 < D.ne);
  };
  if (has_face(blockIdx.x, threadIdx.x)) {
    const int inf = D.ef_info[(size_t)(listed ? elist[blockIdx.x] : blockIdx.x * EPB) * 6 +
                              threadIdx.x];
    s_ef[0][threadIdx.x] = inf;
    s_si[0][threadIdx.x] = reinterpret_cast<const int4*>(D.side_info)[inf >> 3];
  }
  __syncthreads();
  if (threadIdx.x == 0 && (int)blockIdx.x < ngroups) {
    issue_ja(blockIdx.x);
    issue_f(blockIdx.x, 0);
  }

  int it = 0;
  bool gated = GT.n == 0;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    const int nxt = grp + gridDim.x;
    const int cb = it & 1, nbuf = cb ^ 1;
    if (!gated && grp >= GT.pos) {   // the halo traces of the listed boundary elements
      gate_wait(GT);
      gated = true;
    }
    const int e = listed ? elist[grp] : grp * EPB + le;
    const bool active = (le < EPB) && (e < D.ne);
    // next group's ef_info (its side records follow once these have landed)
    const bool tab = has_face(nxt, threadIdx.x);
    if (tab)
      cp_async4(&s_ef[nbuf][threadIdx.x],
                D.ef_info + (size_t)(listed ? elist[nxt] : nxt * EPB) * 6 + threadIdx.x);
    // the neighbours' face traces (vstar) are copied into shared memory before the
    // TMA waits, so their latency overlaps the wait and the repack (one face node
    // per thread; staged behind the indicator's scratch in w, free at this point)
    constexpr bool kOneFaceNode = 6 * n2 <= n3;
    double* stg = w + 3 * n3 + node * 5;
    int vloc = -1, va = 0, vb = 0, vq = 0, vp = 0, vside = 0, vrep = 0;
    if (VISC && kOneFaceNode && active && node < 6 * n2) {
      vloc = node / n2;
      va = (node % n2) / n1;
      vb = node % n1;
      const int info = s_ef[cb][le * 6 + vloc];
      vside = info >> 3;
      vrep = (info >> 2) & 1;
      orient<N>(info & 3, va, vb, vp, vq);
      const double* src = trace_ptr<N>(D, U, s_si[cb][le * 6 + vloc], vside, 1 - vrep, vq, vp);
#pragma unroll
      for (int v = 0; v < 5; ++v) cp_async8(stg + v, src + v);
    }
    mbar_wait(&bar[1], it & 1);
    mbar_wait(&bar[0], it & 1);
    const double* ub = sU + s_off[EPB * 14 + 1] + le * n3 * 5;
    const double* ja = sJ + s_off[EPB * 14] + le * n3 * 9;
    const double* ij = sIJ + le * DM::IJB + s_off[le * 14 + 13];
    const double hs = SPLIT ? 0.5 : 1.0;   // split form: prims / metrics stored halved
    double pr[7], rhoE = 0.0;
    if (active) {
      double u[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) u[v] = ub[node * 5 + v];
      prim_point(u, pr, G);
      if (pr[0] <= 0.0 || pr[4] <= 0.0) atomicOr(&D.status[HDG_STATUS_BAD_PRIM], 1);
      rhoE = u[4];
      if (P.shock && P.indicator == 0) {
        // rho * p with the indicator's own pressure formula (src/shock.py:59-63)
        const double ppi = (G.gamma - 1.0) *
                           (u[4] - 0.5 * (u[1] * u[1] + u[2] * u[2] + u[3] * u[3]) / u[0]);
        w[node] = u[0] * ppi;
      }
      Q[pn] = make_double2(hs * pr[0], hs * pr[1]);
      Q[PN + pn] = make_double2(hs * pr[2], hs * pr[3]);
      Q[2 * PN + pn] = make_double2(hs * pr[4], hs * pr[6]);
      Q[3 * PN + pn] = make_double2(hs * pr[5], rhoE);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double* jv = ja + (a * n3 + node) * 3;
        MJ2[a * PN + pn] = make_double2(hs * jv[0], hs * jv[1]);
        MJ1[a * PN + pn] = hs * jv[2];
      }
    }
    if (tab) {
      // the next group's ef_info has landed: fetch the side records it points to
      cp_async_wait_all();
      cp_async16(&s_si[nbuf][threadIdx.x],
                 reinterpret_cast<const int4*>(D.side_info) + (s_ef[nbuf][threadIdx.x] >> 3));
    }
    __syncthreads();
    // raw Ja consumed (repacked): stream the next group's block during this one
    if (threadIdx.x == 0 && nxt < ngroups) issue_ja(nxt);
    if constexpr (elem_work<N, SPLIT, VISC>() >= 3 * n3) {
      if (P.shock) element_indicator<N>(D, P, sb, w, e, active, node);
    }
    double fvo[3][4];   // own contravariant viscous flux (halved for the split form)
    if (VISC) {
      if constexpr (kOneFaceNode) {
        // vstar = mean of both traces' (u,v,w,T) (k_lift_fill); the own trace is this
        // element's boundary node, whose prims are in Q (halved for the split form)
        if (vloc >= 0) {
          cp_async_wait_all();
          double nb[5], pnb[7];
#pragma unroll
          for (int v = 0; v < 5; ++v) nb[v] = stg[v];
          prim_point(nb, pnb, G);
          const int on = pnode<N>(vol_node<N>(vloc, va, vb, (vloc & 1) ? N : 0));
          const double2 q0 = Q[on], q1 = Q[PN + on];
          const double qT = Q[3 * PN + on].x;
          const double sc = SPLIT ? 2.0 : 1.0;   // exact: undoes the halving
          double* o = vs + node * 4;
          o[0] = 0.5 * (sc * q0.y + pnb[1]);
          o[1] = 0.5 * (sc * q1.x + pnb[2]);
          o[2] = 0.5 * (sc * q1.y + pnb[3]);
          o[3] = 0.5 * (sc * qT + pnb[5]);
          if (D.vstar && (!vrep || s_si[cb][le * 6 + vloc].x < 0)) {
            double* dv = D.vstar + ((size_t)vside * n2 + vq * n1 + vp) * 4;
            for (int l = 0; l < 4; ++l) dv[l] = o[l];
          }
        }
      } else {
        if (active) lift_vstar<N, true>(D, U, G, e, node, n3, vs);
      }
      __syncthreads();
      if (active) {
        double g[12];
        const double* fnv = sNV + le * 6 * DM::NVB;
        const double* fss = sSS + le * 6 * DM::SSB;
        const int* foff = s_off + le * 14;
        lift_gradient_packed<N>(D, sb, sD4, MJ2, MJ1, Q, vs, e, node,
                                g, fnv, fss, foff, ij, s_ef[cb] + le * 6);
        const double mu = viscosity(pr[5], G);
        const double lam = conductivity(mu, G);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double fv[5];
          const double2 m2 = MJ2[a * PN + pn];
          viscous_flux_dir(pr[1], pr[2], pr[3], mu, lam, g, m2.x, m2.y, MJ1[a * PN + pn], fv);
#pragma unroll
          for (int v = 0; v < 4; ++v) fvo[a][v] = fv[v + 1];
          if (SPLIT) {
            WF[(a * 2 + 0) * PN + pn] = make_double2(fv[1], fv[2]);
            WF[(a * 2 + 1) * PN + pn] = make_double2(fv[3], fv[4]);
          }
        }
        face_viscous_lgl<N>(D, G, e, node, pr, mu, lam, g, fnv, foff, s_ef[cb] + le * 6,
                            s_si[cb] + le * 6);
      }
      __syncthreads();
    }
    // U, 1/J and the side blocks of this group are consumed: stream the next group's
    if (threadIdx.x == 0 && nxt < ngroups) issue_f(nxt, nbuf);
    double ut[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (SPLIT) {
      if (active) {
        // k_vol_int_split (:142-209): ascending-alpha sums of Dsplit F# per direction
        const double* DsT = sDsT;
        const double hr = 0.5 * pr[0], hu = 0.5 * pr[1], hv = 0.5 * pr[2], hw = 0.5 * pr[3],
                     hp = 0.5 * pr[4], hh = 0.5 * pr[6];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const int m = d == 0 ? i : (d == 1 ? j : k);
          const int pstride = d == 0 ? 1 : (d == 1 ? n1 + kXiPad<N> : n1 * (n1 + kXiPad<N>));
          const int pbase = pn - m * pstride;
          const double2 mo = MJ2[d * PN + pn];
          const double jxm = mo.x, jym = mo.y, jzm = MJ1[d * PN + pn];
          double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
          double dsum = 0.0;   // fast set: row sum of Dsplit for the own viscous half
#pragma unroll
          for (int al = 0; al < n1; ++al) {
            const int pa = pbase + al * pstride;
            const double2 q0 = Q[pa], q1 = Q[PN + pa], q2 = Q[2 * PN + pa];
            const double2 ma = MJ2[d * PN + pa];
            const double dma = DsT[al * n1 + m];
            if constexpr (kExact) {
              double fs[5];
              kep_flux_half(hr, hu, hv, hw, hp, hh, q0.x, q0.y, q1.x, q1.y, q2.x, q2.y,
                            jxm + ma.x, jym + ma.y, jzm + MJ1[d * PN + pa], fs);
              if (VISC) {
                // the reference adds the viscous mean inside the two-point flux
                const double2 w0 = WF[(d * 2 + 0) * PN + pa], w1 = WF[(d * 2 + 1) * PN + pa];
                fs[1] += fvo[d][0] + w0.x;
                fs[2] += fvo[d][1] + w0.y;
                fs[3] += fvo[d][2] + w1.x;
                fs[4] += fvo[d][3] + w1.y;
              }
#pragma unroll
              for (int v = 0; v < 5; ++v) acc[v] += dma * fs[v];
            } else {
              kep_acc(hr, hu, hv, hw, hp, hh, q0, q1, q2, jxm + ma.x, jym + ma.y,
                      jzm + MJ1[d * PN + pa], dma, acc);
              if (VISC) {
                // linear part split off: sum_a D (f_m + f_a)/2 = f_m/2 sum_a D + sum_a D f_a/2
                const double2 w0 = WF[(d * 2 + 0) * PN + pa], w1 = WF[(d * 2 + 1) * PN + pa];
                acc[1] = fma(dma, w0.x, acc[1]);
                acc[2] = fma(dma, w0.y, acc[2]);
                acc[3] = fma(dma, w1.x, acc[3]);
                acc[4] = fma(dma, w1.y, acc[4]);
                dsum += dma;
              }
            }
          }
          if (VISC && !kExact) {
            // own flux re-read from WF (bitwise fvo): fvo needs no registers in the fast set
            const double2 f0 = WF[(d * 2 + 0) * PN + pn], f1 = WF[(d * 2 + 1) * PN + pn];
            acc[1] = fma(dsum, f0.x, acc[1]);
            acc[2] = fma(dsum, f0.y, acc[2]);
            acc[3] = fma(dsum, f1.x, acc[3]);
            acc[4] = fma(dsum, f1.y, acc[4]);
          }
#pragma unroll
          for (int v = 0; v < 5; ++v) ut[v] += acc[v];
        }
      }
    } else {
      // k_vol_int_standard (:109-139)
      if (active) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double2 m2 = MJ2[a * PN + pn];
          double f[5];
          euler_flux_dir(pr[0], pr[1], pr[2], pr[3], pr[4], rhoE, m2.x, m2.y, MJ1[a * PN + pn], f);
          if (VISC) {
#pragma unroll
            for (int v = 1; v < 5; ++v) f[v] += fvo[a][v - 1];
          }
#pragma unroll
          for (int v = 0; v < 5; ++v) w[(a * 5 + v) * n3 + node] = f[v];
        }
      }
      __syncthreads();
      if (active) {
        const double* Dh = sb + DM::oDhat;
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          double acc = 0.0;
          for (int al = 0; al < n1; ++al)
            acc += Dh[i * n1 + al] * w[(0 * 5 + v) * n3 + k * n2 + j * n1 + al] +
                   Dh[j * n1 + al] * w[(1 * 5 + v) * n3 + k * n2 + al * n1 + i] +
                   Dh[k * n1 + al] * w[(2 * 5 + v) * n3 + al * n2 + j * n1 + i];
          ut[v] += acc;
        }
      }
    }
    if (active) {
      double* dst = D.vol + ((size_t)e * n3 + node) * 5;
#pragma unroll
      for (int v = 0; v < 5; ++v) dst[v] = ut[v];
    }
    if (tab) cp_async_wait_all();   // the next group's side records
    __syncthreads();   // Q / MJ / vs / w are free for the next group
  }
}

// C: per node, Ut = -(1/J)(Vol + gather SurfInt) [+ MMS source], then store Ut or
// the LSERK update (timedisc.py:132-137 without FMA contraction). DT (the last
// stage of a step): the next step's k_local_dt + isfinite on the updated U, so
// the per-step dt pass over U / Ja / J needs no kernel of its own.
template <int N, bool DT>
__device__ __forceinline__ void update_node(const hdg_domain& D, const hdg_params& P,
                                            const VolArgs& V, const int32_t* __restrict__ elist,
                                            const Gate& GT, long tt, unsigned long long& dtbits,
                                            int& nonfinite) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3;
  const int e = elist ? elist[tt / n3] : (int)(tt / n3), node = (int)(tt % n3);
  const long t = (long)e * n3 + node;
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  const size_t o = (size_t)t * 5;
  const int vmode = V.mode & 15;
  const bool lserk = vmode != HDG_MODE_STORE_UT;
  // every streaming load is issued before the gather (memory-level parallelism):
  // Vol and 1/J (read once: evict-first) and, for the stage update, U and dU
  double ut[5], uo[5], dprev[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) ut[v] = __ldcs(D.vol + o + v);
  const double wj = -__ldcs(D.invJ + t);
  if (lserk) {
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      uo[v] = V.U[o + v];
      dprev[v] = vmode == HDG_MODE_LSERK ? V.out[o + v] : 0.0;
    }
  }
#pragma unroll
  for (int loc = 0; loc < 6; ++loc) {
    int m, a, b;
    face_coords(loc >> 1, i, j, k, m, a, b);
    if (m != ((loc & 1) ? N : 0)) continue;
    const int info = D.ef_info[e * 6 + loc];
    const int s = info >> 3, code = info & 3;
    const double sign = ((info >> 2) & 1) ? -1.0 : 1.0;
    const double wt = sign * D.basis[((loc & 1) ? DM::oLhp : DM::oLhm) + m];
    int p, qq;
    orient<N>(code, a, b, p, qq);
    const double* fs = D.fstar + ((size_t)s * n2 + qq * n1 + p) * 5;
#pragma unroll
    // a gated launch reads halo rows written over NVLink during the kernel: L2 only
    for (int v = 0; v < 5; ++v) ut[v] += wt * (GT.n ? __ldcg(fs + v) : fs[v]);
  }
#pragma unroll
  for (int v = 0; v < 5; ++v) ut[v] *= wj;
  if (P.shock) {
    // FV subcell blend after ApplyJac (k_blend, src/shock.py:198-210)
    const double a = D.alpha[e];
    if (a > 0.0) {
      const double b = 1.0 - a;
      const double* rf = D.rfv + o;
#pragma unroll
      for (int v = 0; v < 5; ++v) ut[v] = b * ut[v] + a * rf[v];
    }
  }
  const double tstage = V.time ? V.time[0] + V.c * V.time[1] : V.t_host;
  if (P.source) add_mms_source(P, D.x + (size_t)t * 3, tstage, ut);
  if (!lserk) {
#pragma unroll
    for (int v = 0; v < 5; ++v) V.out[o + v] = ut[v];
  } else {
    const double dt = V.time[1];
    double un[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const double du = vmode == HDG_MODE_LSERK_FIRST
                            ? __dmul_rn(dt, ut[v])
                            : __dadd_rn(__dmul_rn(dprev[v], V.A), __dmul_rn(dt, ut[v]));
      V.out[o + v] = du;
      un[v] = __dadd_rn(uo[v], __dmul_rn(V.B, du));
      V.U[o + v] = un[v];
    }
    if constexpr (DT) {
      // the next step's _compute_dt on the new state (src/parallel.py:595-604)
#pragma unroll
      for (int v = 0; v < 5; ++v) nonfinite |= !isfinite(un[v]);
      const Gas G = make_gas(P);
      const double best = node_dt<N>(un, D, P, G, e, node, D.J[t], P.cfl, P.cfl_visc);
      if (best >= 0.0) dtbits = (unsigned long long)__double_as_longlong(best);
    }
  }
}

template <int N, bool DT>
__global__ void __launch_bounds__(256) update_kernel(hdg_domain D, hdg_params P, VolArgs V,
                                                     const int32_t* __restrict__ elist, int nlist,
                                                     Gate GT) {
  constexpr int n3 = Dim<N>::n3;
  const long tt = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long nn = elist ? (long)nlist * n3 : (long)D.ne * n3;
  if (GT.n) {
    // elements at list position >= GT.pos read f* a neighbour rank computed
    const long last = min((long)(blockIdx.x + 1) * blockDim.x, nn) - 1;
    if (last / n3 >= GT.pos) gate_wait(GT);
  }
  unsigned long long dtbits = 0x7ff0000000000000ULL;   // +inf
  int nonfinite = 0;
  if (tt < nn) update_node<N, DT>(D, P, V, elist, GT, tt, dtbits, nonfinite);
  else if (!DT) return;
  // one call site for every thread of the block (warp shuffles + barrier inside)
  if constexpr (DT) reduce_dt_block(D, dtbits, nonfinite);
}
