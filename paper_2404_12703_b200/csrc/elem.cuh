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
// stream. Each A block prefetches the element one resident wave ahead into L2
// with cp.async.bulk.prefetch.L2 so HBM traffic overlaps the FP64 work.

__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  // 16-byte aligned start, size a multiple of 16 (the hint never faults)
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  bytes = (bytes + 31u) & ~15u;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
}

template <int N, bool SPLIT, bool VISC>
__host__ __device__ constexpr int elem_work() {
  using DM = Dim<N>;
  // split: per-direction viscous flux rows for all 3 directions (12 rows)
  // standard: the 15 contravariant flux rows
  return SPLIT ? (VISC ? 12 * DM::n3 : 0) : 15 * DM::n3;
}

template <int N, bool SPLIT, bool VISC>
__global__ void __launch_bounds__(Dim<N>::THREADS, 1)
    elem_kernel(hdg_domain D, hdg_params P, const double* __restrict__ U, int wave) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3, EPB = DM::EPB;
  extern __shared__ double smem[];
  double* sb = smem;
  double* sq = sb + ((DM::BASIS + 1) & ~1);              // [EPB][8][n3] rho u v w p h T rhoE
  double* sja = sq + EPB * 8 * n3;                       // [EPB][9*n3] raw Ja block
  double* svs = sja + EPB * 9 * n3;                      // [EPB][6*n2*4] (VISC)
  double* sw = svs + (VISC ? EPB * 24 * n2 : 0);         // [EPB][elem_work]
  const int le = threadIdx.x / n3;
  const int node = threadIdx.x % n3;
  const int e = blockIdx.x * EPB + le;
  const bool active = (le < EPB) && (e < D.ne);
  if (threadIdx.x < EPB && wave > 0) {
    const int en = (blockIdx.x + wave) * EPB + threadIdx.x;
    if (en < D.ne) {
      l2_prefetch(U + (size_t)en * n3 * 5, n3 * 5 * 8);
      l2_prefetch(D.Ja + (size_t)en * n3 * 9, n3 * 9 * 8);
      l2_prefetch(D.invJ + (size_t)en * n3, n3 * 8);
    }
  }
  load_basis<N>(sb, D.basis);
  const Gas G = make_gas(P);
  double* q = sq + le * 8 * n3;
  double* ja = sja + le * 9 * n3;
  double* vs = svs + le * 24 * n2;
  double* w = sw + le * elem_work<N, SPLIT, VISC>();
  double pr[7], rhoE = 0.0;
  if (active) {
    double u[5];
    const double* src = U + ((size_t)e * n3 + node) * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = src[v];
    prim_point(u, pr, G);
    if (pr[0] <= 0.0 || pr[4] <= 0.0) atomicOr(&D.status[HDG_STATUS_BAD_PRIM], 1);
    rhoE = u[4];
    q[0 * n3 + node] = pr[0];
    q[1 * n3 + node] = pr[1];
    q[2 * n3 + node] = pr[2];
    q[3 * n3 + node] = pr[3];
    q[4 * n3 + node] = pr[4];
    q[5 * n3 + node] = pr[6];
    q[6 * n3 + node] = pr[5];
    q[7 * n3 + node] = rhoE;
    const double* jsrc = D.Ja + (size_t)e * 9 * n3;
    for (int t = node; t < 9 * n3; t += n3) ja[t] = jsrc[t];
  }
  __syncthreads();
  double fvo[3][4];   // own contravariant viscous flux, a = 0..2, v = 1..4
  if (VISC) {
    if (active) lift_vstar<N, true>(D, U, G, e, node, n3, vs);
    __syncthreads();
    if (active) {
      double g[12];
      lift_gradient<N, true>(D, sb, ja, q + n3, q + 6 * n3, vs, e, node, g);
      const double mu = viscosity(pr[5], G);
      const double lam = conductivity(mu, G);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double fv[5];
        const double* jv = ja + (a * n3 + node) * 3;
        viscous_flux_dir(pr[1], pr[2], pr[3], mu, lam, g, jv[0], jv[1], jv[2], fv);
#pragma unroll
        for (int v = 0; v < 4; ++v) fvo[a][v] = fv[v + 1];
        if (SPLIT) {
#pragma unroll
          for (int v = 0; v < 4; ++v) w[(a * 4 + v) * n3 + node] = fv[v + 1];
        }
      }
      face_viscous_lgl<N>(D, G, e, node, pr, mu, lam, g);
    }
  }
  double ut[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  if (SPLIT) {
    if (VISC) __syncthreads();
    if (active) {
      // k_vol_int_split (:142-209): ascending-alpha sums of Dsplit F# per direction
      const double* Ds = sb + DM::oDsplit;
#pragma unroll 1
      for (int d = 0; d < 3; ++d) {
        const int m = d == 0 ? i : (d == 1 ? j : k);
        const int stride = d == 0 ? 1 : (d == 1 ? n1 : n2);
        const int base = node - m * stride;
        const double* jd = ja + d * n3 * 3;
        const double jxm = jd[node * 3 + 0], jym = jd[node * 3 + 1], jzm = jd[node * 3 + 2];
        double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int al = 0; al < n1; ++al) {
          const int na = base + al * stride;
          double fs[5];
          kep_flux(pr[0], pr[1], pr[2], pr[3], pr[4], pr[6], q[0 * n3 + na], q[1 * n3 + na],
                   q[2 * n3 + na], q[3 * n3 + na], q[4 * n3 + na], q[5 * n3 + na],
                   0.5 * (jxm + jd[na * 3 + 0]), 0.5 * (jym + jd[na * 3 + 1]),
                   0.5 * (jzm + jd[na * 3 + 2]), fs);
          if (VISC) {
            const double* wf = w + d * 4 * n3;
#pragma unroll
            for (int v = 1; v < 5; ++v)
              fs[v] += 0.5 * (wf[(v - 1) * n3 + node] + wf[(v - 1) * n3 + na]);
          }
          const double dma = Ds[m * n1 + al];
#pragma unroll
          for (int v = 0; v < 5; ++v) acc[v] += dma * fs[v];
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
        const double* jv = ja + (a * n3 + node) * 3;
        double f[5];
        euler_flux_dir(pr[0], pr[1], pr[2], pr[3], pr[4], rhoE, jv[0], jv[1], jv[2], f);
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
}

// C: per node, Ut = -(1/J)(Vol + gather SurfInt) [+ MMS source], then store Ut or
// the LSERK update (timedisc.py:132-137 without FMA contraction).
template <int N>
__global__ void __launch_bounds__(256) update_kernel(hdg_domain D, hdg_params P, VolArgs V) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)D.ne * n3) return;
  const int e = (int)(t / n3), node = (int)(t % n3);
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  const size_t o = (size_t)t * 5;
  double ut[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) ut[v] = D.vol[o + v];
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
    for (int v = 0; v < 5; ++v) ut[v] += wt * fs[v];
  }
  const double wj = -D.invJ[t];
#pragma unroll
  for (int v = 0; v < 5; ++v) ut[v] *= wj;
  const double tstage = V.time ? V.time[0] + V.c * V.time[1] : V.t_host;
  if (P.source) add_mms_source(P, D.x + (size_t)t * 3, tstage, ut);
  const int vmode = V.mode & 15;
  if (vmode == HDG_MODE_STORE_UT) {
#pragma unroll
    for (int v = 0; v < 5; ++v) V.out[o + v] = ut[v];
  } else {
    const double dt = V.time[1];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const double du = vmode == HDG_MODE_LSERK_FIRST
                            ? __dmul_rn(dt, ut[v])
                            : __dadd_rn(__dmul_rn(V.out[o + v], V.A), __dmul_rn(dt, ut[v]));
      V.out[o + v] = du;
      V.U[o + v] = __dadd_rn(V.U[o + v], __dmul_rn(V.B, du));
    }
  }
}
