// DGSEM hot-path kernels for sm_100a (FP64). Included twice by kernels_exact.cu
// (-fmad=false) and kernels_fast.cu (FMA contraction), each inside its own
// namespace, so one source gives a bit-exact and a fast kernel set.
//
// Kernel map (reference kernels they replace, src/operator.py unless noted):
//   lift_kernel    k_lift_fill + k_lift_volume + k_lift_surf_and_jac + k_viscous_contravariant
//                  + k_prolong_grad + the face half of k_fill_flux_viscous, fused per element
//   flux_kernel    k_fill_flux_convective + k_fill_flux_viscous (mean of the element-side
//                  viscous face fluxes), per face node; LGL traces gathered straight from U
//   volume_kernel  k_cons_to_prim + k_vol_int_split | k_vol_int_standard + k_surf_int +
//                  k_apply_jac + k_indicator + k_fv_residual + k_blend (src/shock.py) +
//                  k_mms_source (src/testcases.py) + the LSERK stage (src/timedisc.py:132-137)
//   prolong_kernel k_prolong / apply_bc_traces (API + GL path)
//   dt_kernel      k_local_dt + isfinite(U) (src/parallel.py:595-604)
// (included inside a namespace after common.cuh; see kernels_exact.cu)

template <int N>
struct Dim {
  static constexpr int n1 = N + 1, n2 = n1 * n1, n3 = n2 * n1;
  // elements per CTA so that a CTA has >= ~128 node-threads
  static constexpr int EPB = (n3 >= 100) ? 1 : ((128 + n3 - 1) / n3);
  static constexpr int THREADS = ((EPB * n3 + 31) / 32) * 32;
  static constexpr int BASIS = 4 * n2 + 6 * n1;
  // shared-memory slots of per-side / per-element blocks staged by TMA (+ slack
  // for a 16-byte aligned superset, rounded to 16-byte multiples)
  static constexpr int NVB = (n2 * 3 + 3) & ~1, SSB = (n2 + 3) & ~1, IJB = (n3 + 3) & ~1;
  // packed basis offsets
  static constexpr int oD = 0, oDhat = n2, oDsplit = 2 * n2, oVinv = 3 * n2, oW = 4 * n2,
                       oLm = 4 * n2 + n1, oLp = 4 * n2 + 2 * n1, oLhm = 4 * n2 + 3 * n1,
                       oLhp = 4 * n2 + 4 * n1, oIW = 4 * n2 + 5 * n1;
};

// volume node of face-tangential point (a, b) at normal index n (_vol_index, :33-41)
template <int N>
__device__ __forceinline__ int vol_node(int loc, int a, int b, int n) {
  constexpr int n1 = N + 1, n2 = n1 * n1;
  const int d = loc >> 1;
  if (d == 0) return b * n2 + a * n1 + n;   // (i,j,k) = (n,a,b)
  if (d == 1) return a * n2 + n * n1 + b;   // (b,n,a)
  return n * n2 + b * n1 + a;               // (a,b,n)
}

// _orient (:44-52); involution
template <int N>
__device__ __forceinline__ void orient(int code, int a, int b, int& p, int& q) {
  p = (code & 1) ? N - a : a;
  q = (code & 2) ? N - b : b;
}

// (m, a, b) of node (i,j,k) w.r.t. the normal axis d (k_surf_int, :347-353)
__device__ __forceinline__ void face_coords(int d, int i, int j, int k, int& m, int& a, int& b) {
  if (d == 0) { m = i; a = j; b = k; }
  else if (d == 1) { m = j; a = k; b = i; }
  else { m = k; a = i; b = j; }
}

template <int N>
__device__ __forceinline__ void load_basis(double* sb, const double* g) {
  for (int t = threadIdx.x; t < Dim<N>::BASIS; t += blockDim.x) sb[t] = g[t];
}

__device__ __forceinline__ void side_decode(int meta, int& loc_p, int& loc_r, int& code, int& bc,
                                            int& kind) {
  loc_p = meta & 7;
  loc_r = (meta >> 3) & 7;
  code = (meta >> 6) & 3;
  bc = (meta >> 8) & 15;
  kind = meta >> 12;
}

// ---------------------------------------------------------------------------
// trace of one role of a side at storage point (q, p)
//   role 0 = primary ("L"), role 1 = replica ("R").
// LGL with a local element: the trace is the element's boundary node (prolong
// is an exact copy, tests/test_operator.py:84-96). Otherwise (GL, or the
// element lives on another rank) it is read from the UL/UR trace arrays.
template <int N, bool LGL>
__device__ __forceinline__ void load_trace(const hdg_domain& D, const double* __restrict__ U,
                                           int s, int role, int q, int p, double out[5]) {
  constexpr int n1 = N + 1, n2 = n1 * n1, n3 = n2 * n1;
  const int4 si = reinterpret_cast<const int4*>(D.side_info)[s];
  int loc_p, loc_r, code, bc, kind;
  side_decode(si.z, loc_p, loc_r, code, bc, kind);
  if (role == 1 && kind == HDG_SIDE_BC) {
#pragma unroll
    for (int v = 0; v < 5; ++v) out[v] = D.bc_states[bc * 5 + v];
    return;
  }
  const int e = role == 0 ? si.x : si.y;
  if (LGL && e >= 0) {
    int node;
    if (role == 0) {
      node = vol_node<N>(loc_p, p, q, (loc_p & 1) ? N : 0);
    } else {
      int a, b;
      orient<N>(code, p, q, a, b);
      node = vol_node<N>(loc_r, a, b, (loc_r & 1) ? N : 0);
    }
    const double* src = U + ((size_t)e * n3 + node) * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) out[v] = src[v];
  } else {
    // UL/UR rows (GL traces, or a neighbour rank's halo written over NVLink):
    // L2-coherent loads, never a stale L1 line
    const double* src = (role == 0 ? D.UL : D.UR) + ((size_t)s * n2 + q * n1 + p) * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) out[v] = __ldcg(src + v);
  }
}

// address of the same trace (LGL) given the side record si of side s, so that
// the caller can copy it asynchronously
template <int N>
__device__ __forceinline__ const double* trace_ptr(const hdg_domain& D, const double* U, int4 si,
                                                   int s, int role, int q, int p) {
  constexpr int n1 = N + 1, n2 = n1 * n1, n3 = n2 * n1;
  int loc_p, loc_r, code, bc, kind;
  side_decode(si.z, loc_p, loc_r, code, bc, kind);
  if (role == 1 && kind == HDG_SIDE_BC) return D.bc_states + bc * 5;
  const int e = role == 0 ? si.x : si.y;
  if (e >= 0) {
    int node;
    if (role == 0) {
      node = vol_node<N>(loc_p, p, q, (loc_p & 1) ? N : 0);
    } else {
      int a, b;
      orient<N>(code, p, q, a, b);
      node = vol_node<N>(loc_r, a, b, (loc_r & 1) ? N : 0);
    }
    return U + ((size_t)e * n3 + node) * 5;
  }
  return (role == 0 ? D.UL : D.UR) + ((size_t)s * n2 + q * n1 + p) * 5;
}

// ---------------------------------------------------------------------------
// surface flux: one thread per (listed side, q, p)
template <int N, bool LGL, bool VISC>
__global__ void __launch_bounds__(64, (VISC ? 16 : 20)) flux_kernel(hdg_domain D, hdg_params P,
                                                   const double* __restrict__ U,
                                                   const int32_t* __restrict__ sides, int nsides,
                                                   int solver, int from_arrays, Gate GT) {
  constexpr int n1 = N + 1, n2 = n1 * n1;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (GT.n) {
    // sides at list position >= GT.pos need the neighbours' face payload
    const long last = min((long)(blockIdx.x + 1) * blockDim.x, (long)nsides * n2) - 1;
    if (last / n2 >= GT.pos) gate_wait(GT);
  }
  if (t >= (long)nsides * n2) return;
  const int s = sides ? sides[t / n2] : (int)(t / n2);   // NULL: all sides, no indirection
  const int fq = (int)(t % n2);
  const int q = fq / n1, p = fq % n1;
  const Gas G = make_gas(P);
  const size_t fo = (size_t)s * n2 + fq;
  // side geometry and (viscous) the element-side face fluxes are independent of
  // the traces: issue their loads first
  const double* nv = D.nvec + fo * 3;
  const double nx = nv[0], ny = nv[1], nz = nv[2], ss = D.ssurf[fo];
  double fvl[4], fvr[4];
  if (VISC) {
    const double* fl = D.fvface + (((size_t)s * 2 + 0) * n2 + fq) * 4;
    const double* fr = D.fvface + (((size_t)s * 2 + 1) * n2 + fq) * 4;
#pragma unroll
    for (int v = 0; v < 4; ++v) {   // gated: the replica half arrives over NVLink in-kernel
      fvl[v] = GT.n ? __ldcg(fl + v) : fl[v];
      fvr[v] = GT.n ? __ldcg(fr + v) : fr[v];
    }
  }
  double uL[5], uR[5], pl[7], pr[7], f[5];
  if (from_arrays) {
    load_trace<N, false>(D, U, s, 0, q, p, uL);
    load_trace<N, false>(D, U, s, 1, q, p, uR);
  } else {
    load_trace<N, LGL>(D, U, s, 0, q, p, uL);
    load_trace<N, LGL>(D, U, s, 1, q, p, uR);
  }
  prim_point(uL, pl, G);
  prim_point(uR, pr, G);
  if (pl[0] <= 0.0 || pl[4] <= 0.0 || pr[0] <= 0.0 || pr[4] <= 0.0)
    atomicMax(&D.status[HDG_STATUS_BAD_SIDE], s);
  riemann(solver, pl, uL[4], pr, uR[4], nx, ny, nz, G.gamma, f);
  double* out = D.fstar + fo * 5;
#pragma unroll
  for (int v = 0; v < 5; ++v) f[v] = f[v] * ss;
  if (VISC) {
#pragma unroll
    for (int v = 1; v < 5; ++v) f[v] = f[v] + 0.5 * (fvl[v - 1] + fvr[v - 1]) * ss;
  }
#pragma unroll
  for (int v = 0; v < 5; ++v) out[v] = f[v];
}

// ---------------------------------------------------------------------------
// prolong (k_prolong): thread per (row, a, b)
template <int N>
__global__ void __launch_bounds__(256) prolong_kernel(hdg_domain D, const double* __restrict__ U,
                                                      const int32_t* __restrict__ rows, int nrows) {
  constexpr int n1 = N + 1, n2 = n1 * n1, n3 = n2 * n1;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)nrows * n2) return;
  const int r = (int)(t / n2), ab = (int)(t % n2);
  const int a = ab / n1, b = ab % n1;
  const int s = rows[r * 5 + 0], e = rows[r * 5 + 1], loc = rows[r * 5 + 2];
  const int is_p = rows[r * 5 + 3], code = rows[r * 5 + 4];
  const double* lv = D.basis + ((loc & 1) ? Dim<N>::oLp : Dim<N>::oLm);
  int p, q;
  orient<N>(code, a, b, p, q);
  const double* ue = U + (size_t)e * n3 * 5;
  double* dst = (is_p ? D.UL : D.UR) + ((size_t)s * n2 + q * n1 + p) * 5;
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    double acc = 0.0;
    for (int m = 0; m < n1; ++m) acc += lv[m] * ue[vol_node<N>(loc, a, b, m) * 5 + v];
    dst[v] = acc;
  }
}

__global__ void bc_traces_kernel(hdg_domain D, const int32_t* __restrict__ sides, int nsides,
                                 int n2) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)nsides * n2 * 5) return;
  const int v = (int)(t % 5);
  const long sp = t / 5;
  const int s = sides[sp / n2];
  const int bc = (reinterpret_cast<const int4*>(D.side_info)[s].z >> 8) & 15;
  D.UR[((size_t)s * n2 + sp % n2) * 5 + v] = D.bc_states[bc * 5 + v];
}

// ---------------------------------------------------------------------------
// BR1 lifting building blocks (shared by lift_kernel and elem_kernel)

// central lifting flux vstar on the element's 6 faces, element face coords
// (k_lift_fill, :377-391); vs[(loc*n2 + a*n1 + b)*4 + l]
template <int N, bool LGL>
__device__ __forceinline__ void lift_vstar(const hdg_domain& D, const double* __restrict__ U,
                                           const Gas& G, int e, int tid, int nthreads, double* vs) {
  constexpr int n1 = N + 1, n2 = n1 * n1;
  for (int t = tid; t < 6 * n2; t += nthreads) {
    const int loc = t / n2, ab = t % n2, a = ab / n1, b = ab % n1;
    const int info = D.ef_info[e * 6 + loc];
    const int s = info >> 3, rep = (info >> 2) & 1, code = info & 3;
    int p, q;
    orient<N>(code, a, b, p, q);
    double uo[5], un[5], po[7], pn[7];
    load_trace<N, LGL>(D, U, s, rep, q, p, uo);
    load_trace<N, LGL>(D, U, s, 1 - rep, q, p, un);
    prim_point(uo, po, G);
    prim_point(un, pn, G);
    double* o = vs + t * 4;
    o[0] = 0.5 * (po[1] + pn[1]);
    o[1] = 0.5 * (po[2] + pn[2]);
    o[2] = 0.5 * (po[3] + pn[3]);
    o[3] = 0.5 * (po[5] + pn[5]);
    if (D.vstar) {
      const int4 si = reinterpret_cast<const int4*>(D.side_info)[s];
      if (!rep || si.x < 0) {
        double* dv = D.vstar + ((size_t)s * n2 + q * n1 + p) * 4;
        for (int l = 0; l < 4; ++l) dv[l] = o[l];
      }
    }
  }
}

// lifted gradient g[d*4+l] at node (i,j,k): weak volume term (k_lift_volume,
// :394-418), surface term and 1/J (k_lift_surf_and_jac, :421-453).
// ja: raw Ja block [a][node][c]; pu: u,v,w rows (stride n3); pT: T row.
// Dh: the weak derivative matrix Dhat, or 4*Dhat when ja and pu/pT hold halved
// values (elem_kernel): (4D)(Ja/2)(phi/2) == D Ja phi exactly, term by term.
// fnv/fss/foff: this element's staged nvec / ssurf side blocks in shared memory
// (slot loc, word offsets foff[2 loc], foff[2 loc + 1]) and fij its staged 1/J,
// or nullptr to read global memory.
template <int N, bool LGL>
__device__ __forceinline__ void lift_gradient(const hdg_domain& D, const double* sb,
                                              const double* Dh, const double* ja,
                                              const double* pu, const double* pT,
                                              const double* vs, int e, int node, double g[12],
                                              const double* fnv = nullptr,
                                              const double* fss = nullptr,
                                              const int* foff = nullptr,
                                              const double* fij = nullptr) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3;
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
#pragma unroll
  for (int c = 0; c < 12; ++c) g[c] = 0.0;
  for (int al = 0; al < n1; ++al) {
    const double di = Dh[i * n1 + al], dj = Dh[j * n1 + al], dk = Dh[k * n1 + al];
    const int ni = k * n2 + j * n1 + al, nj = k * n2 + al * n1 + i, nk = al * n2 + j * n1 + i;
    const double phi_i[4] = {pu[ni], pu[n3 + ni], pu[2 * n3 + ni], pT[ni]};
    const double phi_j[4] = {pu[nj], pu[n3 + nj], pu[2 * n3 + nj], pT[nj]};
    const double phi_k[4] = {pu[nk], pu[n3 + nk], pu[2 * n3 + nk], pT[nk]};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double jai = di * ja[(0 * n3 + ni) * 3 + d];
      const double jaj = dj * ja[(1 * n3 + nj) * 3 + d];
      const double jak = dk * ja[(2 * n3 + nk) * 3 + d];
#pragma unroll
      for (int l = 0; l < 4; ++l) g[d * 4 + l] += jai * phi_i[l] + jaj * phi_j[l] + jak * phi_k[l];
    }
  }
#pragma unroll
  for (int loc = 0; loc < 6; ++loc) {
    const int d = loc >> 1;
    int m, a, b;
    face_coords(d, i, j, k, m, a, b);
    if (LGL && m != ((loc & 1) ? N : 0)) continue;   // lhat is exactly 0 off the face
    const int info = D.ef_info[e * 6 + loc];
    const int s = info >> 3, code = info & 3;
    const double sign = ((info >> 2) & 1) ? -1.0 : 1.0;
    const double lh = sb[((loc & 1) ? DM::oLhp : DM::oLhm) + m];
    int p, q;
    orient<N>(code, a, b, p, q);
    const int fq = q * n1 + p;
    const double* nvp;
    double ssv;
    if (fnv) {
      nvp = fnv + loc * DM::NVB + foff[2 * loc] + fq * 3;
      ssv = fss[loc * DM::SSB + foff[2 * loc + 1] + fq];
    } else {
      nvp = D.nvec + ((size_t)s * n2 + fq) * 3;
      ssv = D.ssurf[(size_t)s * n2 + fq];
    }
    const double w = sign * lh * ssv;
    const double* vsv = vs + (loc * n2 + a * n1 + b) * 4;
#pragma unroll
    for (int dd = 0; dd < 3; ++dd) {
      const double nd = w * nvp[dd];
#pragma unroll
      for (int l = 0; l < 4; ++l) g[dd * 4 + l] += nd * vsv[l];
    }
  }
  const double iw = fij ? fij[node] : D.invJ[(size_t)e * n3 + node];
#pragma unroll
  for (int c = 0; c < 12; ++c) g[c] *= iw;
  if (D.g) {
    double* dg = D.g + ((size_t)e * n3 + node) * 12;
#pragma unroll
    for (int c = 0; c < 12; ++c) dg[c] = g[c];
  }
}

// element-side viscous face fluxes at an LGL boundary node (the per-side half of
// k_fill_flux_viscous, :295-330; the LGL gradient trace is the node value, and
// the Dirichlet ghost uses UR = bc state, gR = gL, :646-649, :704-705)
template <int N>
__device__ __forceinline__ void face_viscous_lgl(const hdg_domain& D, const Gas& G, int e,
                                                 int node, const double pr[7], double mu,
                                                 double lam, const double g[12],
                                                 const double* fnv = nullptr,
                                                 const int* foff = nullptr,
                                                 const int* fef = nullptr,
                                                 const int4* fsi = nullptr) {
  constexpr int n1 = N + 1, n2 = n1 * n1;
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
#pragma unroll
  for (int loc = 0; loc < 6; ++loc) {
    int m, a, b;
    face_coords(loc >> 1, i, j, k, m, a, b);
    if (m != ((loc & 1) ? N : 0)) continue;
    const int info = fef ? fef[loc] : D.ef_info[e * 6 + loc];
    const int s = info >> 3, rep = (info >> 2) & 1, code = info & 3;
    int p, q;
    orient<N>(code, a, b, p, q);
    const int fq = q * n1 + p;
    const double* nv = fnv ? fnv + loc * Dim<N>::NVB + foff[2 * loc] + fq * 3
                           : D.nvec + ((size_t)s * n2 + fq) * 3;
    double fv[5];
    viscous_flux_dir(pr[1], pr[2], pr[3], mu, lam, g, nv[0], nv[1], nv[2], fv);
    double* dst = D.fvface + (((size_t)s * 2 + rep) * n2 + fq) * 4;
#pragma unroll
    for (int v = 1; v < 5; ++v) dst[v - 1] = fv[v];
    if (D.gL) {
      double* dg = (rep ? D.gR : D.gL) + ((size_t)s * n2 + fq) * 12;
#pragma unroll
      for (int c = 0; c < 12; ++c) dg[c] = g[c];
    }
    const int4 si = fsi ? fsi[loc] : reinterpret_cast<const int4*>(D.side_info)[s];
    if (((si.z >> 12) & 3) == HDG_SIDE_BC) {
      const int bc = (si.z >> 8) & 15;
      double ub[5], pb[7];
      for (int v = 0; v < 5; ++v) ub[v] = D.bc_states[bc * 5 + v];
      prim_point(ub, pb, G);
      const double mub = viscosity(pb[5], G);
      const double lamb = conductivity(mub, G);
      viscous_flux_dir(pb[1], pb[2], pb[3], mub, lamb, g, nv[0], nv[1], nv[2], fv);
      double* dr = D.fvface + (((size_t)s * 2 + 1) * n2 + fq) * 4;
#pragma unroll
      for (int v = 1; v < 5; ++v) dr[v - 1] = fv[v];
      if (D.gL) {
        double* dg = D.gR + ((size_t)s * n2 + fq) * 12;
#pragma unroll
        for (int c = 0; c < 12; ++c) dg[c] = g[c];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// BR1 lifting, fused per element (one thread per volume node); GL path and the
// API-level Domain.lift_gradients. The LGL production path is elem_kernel.
template <int N, bool LGL>
__global__ void __launch_bounds__(Dim<N>::THREADS) lift_kernel(hdg_domain D, hdg_params P,
                                                               const double* __restrict__ U) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3, EPB = DM::EPB;
  extern __shared__ double smem[];
  double* sb = smem;                                // basis
  double* sphi = sb + ((DM::BASIS + 1) & ~1);       // [EPB][4][n3]
  double* sja = sphi + EPB * 4 * n3;                // [EPB][9*n3] raw Ja block
  double* svs = sja + EPB * 9 * n3;                 // [EPB][6][n2][4] face vstar (element coords)
  double* sg = svs + EPB * 6 * n2 * 4;              // [EPB][12][n3] (GL only)
  load_basis<N>(sb, D.basis);
  const Gas G = make_gas(P);
  const int le = threadIdx.x / n3;
  const int node = threadIdx.x % n3;
  const int e = blockIdx.x * EPB + le;
  const bool active = (le < EPB) && (e < D.ne);
  double* phi = sphi + le * 4 * n3;
  double* ja = sja + le * 9 * n3;
  double* vs = svs + le * 6 * n2 * 4;
  double pr[7];
  if (active) {
    double u[5];
    const double* src = U + ((size_t)e * n3 + node) * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) u[v] = src[v];
    prim_point(u, pr, G);
    phi[0 * n3 + node] = pr[1];
    phi[1 * n3 + node] = pr[2];
    phi[2 * n3 + node] = pr[3];
    phi[3 * n3 + node] = pr[5];
    const double* jsrc = D.Ja + (size_t)e * 9 * n3;
    for (int t = node; t < 9 * n3; t += n3) ja[t] = jsrc[t];
  }
  __syncthreads();
  if (active) lift_vstar<N, LGL>(D, U, G, e, node, n3, vs);
  __syncthreads();
  double g[12];
  if (active) {
    lift_gradient<N, LGL>(D, sb, sb + DM::oDhat, ja, phi, phi + 3 * n3, vs, e, node, g);
    // contravariant viscous fluxes (k_viscous_contravariant, :89-102)
    const double mu = viscosity(pr[5], G);
    const double lam = conductivity(mu, G);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double fv[5];
      const double* jv = ja + (a * n3 + node) * 3;
      viscous_flux_dir(pr[1], pr[2], pr[3], mu, lam, g, jv[0], jv[1], jv[2], fv);
      double* dst = D.Fvis + ((size_t)e * 3 + a) * 4 * n3 + node;
#pragma unroll
      for (int v = 1; v < 5; ++v) dst[(v - 1) * n3] = fv[v];
    }
    if (LGL) {
      face_viscous_lgl<N>(D, G, e, node, pr, mu, lam, g);
    } else {
      double* gg = sg + le * 12 * n3;
#pragma unroll
      for (int c = 0; c < 12; ++c) gg[c * n3 + node] = g[c];
    }
  }
  if (!LGL) {
    // GL: gradient traces by interpolation (k_prolong_grad, :241-266) and the
    // element-side viscous face flux from the prolonged U trace
    __syncthreads();
    if (active) {
      const double* gg = sg + le * 12 * n3;
      for (int t = node; t < 6 * n2; t += n3) {
        const int loc = t / n2, ab = t % n2, a = ab / n1, b = ab % n1;
        const int info = D.ef_info[e * 6 + loc];
        const int s = info >> 3, rep = (info >> 2) & 1, code = info & 3;
        int p, q;
        orient<N>(code, a, b, p, q);
        const int fq = q * n1 + p;
        const double* lv = sb + ((loc & 1) ? DM::oLp : DM::oLm);
        double gt[12];
#pragma unroll
        for (int c = 0; c < 12; ++c) gt[c] = lv[0] * gg[c * n3 + vol_node<N>(loc, a, b, 0)];
        for (int m = 1; m < n1; ++m) {
          const int nm = vol_node<N>(loc, a, b, m);
#pragma unroll
          for (int c = 0; c < 12; ++c) gt[c] += lv[m] * gg[c * n3 + nm];
        }
        double ut[5], pt[7], fv[5];
        load_trace<N, false>(D, U, s, rep, q, p, ut);
        prim_point(ut, pt, G);
        const double mu = viscosity(pt[5], G);
        const double lam = conductivity(mu, G);
        const double* nv = D.nvec + ((size_t)s * n2 + fq) * 3;
        viscous_flux_dir(pt[1], pt[2], pt[3], mu, lam, gt, nv[0], nv[1], nv[2], fv);
        double* dst = D.fvface + (((size_t)s * 2 + rep) * n2 + fq) * 4;
        for (int v = 1; v < 5; ++v) dst[v - 1] = fv[v];
        if (D.gL) {
          double* dg = (rep ? D.gR : D.gL) + ((size_t)s * n2 + fq) * 12;
          for (int c = 0; c < 12; ++c) dg[c] = gt[c];
        }
        const int4 si = reinterpret_cast<const int4*>(D.side_info)[s];
        if (((si.z >> 12) & 3) == HDG_SIDE_BC) {
          const int bc = (si.z >> 8) & 15;
          double ub[5], pb[7];
          for (int v = 0; v < 5; ++v) ub[v] = D.bc_states[bc * 5 + v];
          prim_point(ub, pb, G);
          const double mub = viscosity(pb[5], G);
          const double lamb = conductivity(mub, G);
          viscous_flux_dir(pb[1], pb[2], pb[3], mub, lamb, gt, nv[0], nv[1], nv[2], fv);
          double* dr = D.fvface + (((size_t)s * 2 + 1) * n2 + fq) * 4;
          for (int v = 1; v < 5; ++v) dr[v - 1] = fv[v];
          if (D.gL) {
            double* dg = D.gR + ((size_t)s * n2 + fq) * 12;
            for (int c = 0; c < 12; ++c) dg[c] = gt[c];
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// the element kernel: volume + surface integral + Jacobian [+ FV blend]
// [+ source] + store Ut / LSERK stage update
// per-element work buffer of the element kernel (doubles): split needs metric (3)
// [+ viscous flux (4)] rows, the standard form 15 flux rows, the FV subcell pass
// one direction of interface fluxes, the indicator 3 modal rows
template <int N, bool SPLIT, bool VISC, bool SHOCK>
__host__ __device__ constexpr int vol_work() {
  using DM = Dim<N>;
  constexpr int work = SPLIT ? (VISC ? 7 * DM::n3 : 3 * DM::n3) : 15 * DM::n3;
  constexpr int fv = SHOCK ? DM::n2 * (DM::n1 + 1) * 5 : 0;
  constexpr int ind = SHOCK ? 3 * DM::n3 : 0;
  constexpr int w1 = work > fv ? work : fv;
  return w1 > ind ? w1 : ind;
}

// k_mms_source (src/testcases.py:51-70) at one node
__device__ __forceinline__ void add_mms_source(const hdg_params& P, const double* xp, double t,
                                               double ut[5]) {
  const double W = 2.0 * 3.141592653589793;
  const double A = P.mms_A, a = P.mms_a, gamma = P.gamma;
  const double c_mom = 0.5 * (5.0 * gamma + 1.0) - a;
  const double c_e1 = A * (3.0 * gamma - a);
  const double c_e2 = 7.5 * gamma + 4.5 - 4.0 * a;
  const double c_e3 = 3.0 * W * gamma * P.mu_ref / P.Pr;
  const double ph = W * (xp[0] + xp[1] + xp[2] - a * t);
  const double sn = sin(ph), cs = cos(ph);
  const double aw = A * W;
  const double s_mom = aw * cs * (2.0 * A * (gamma - 1.0) * sn + c_mom);
  ut[0] += aw * (3.0 - a) * cs;
  ut[1] += s_mom;
  ut[2] += s_mom;
  ut[3] += s_mom;
  ut[4] += aw * (c_e1 * 2.0 * sn * cs + c_e2 * cs + c_e3 * sn);
}

struct VolArgs {
  double* U;            // in (and out for the LSERK modes)
  double* out;          // Ut (mode 0) or dU (modes 1, 2)
  const double* time;   // device [t, dt] or NULL
  double t_host, A, B, c;
  int mode;
};

template <int N, bool SPLIT, bool VISC, bool SHOCK>
__global__ void __launch_bounds__(Dim<N>::THREADS) volume_kernel(hdg_domain D, hdg_params P,
                                                                 VolArgs V) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3, EPB = DM::EPB;
  extern __shared__ double smem[];
  double* sb = smem;
  double* sq = sb + ((DM::BASIS + 1) & ~1);           // [EPB][7][n3]: rho u v w p h rhoE
  constexpr int WORK = vol_work<N, SPLIT, VISC, SHOCK>();
  double* sw = sq + EPB * 7 * n3;                     // work: [EPB][WORK]
  __shared__ double s_alpha[EPB];
  load_basis<N>(sb, D.basis);
  const Gas G = make_gas(P);
  const int le = threadIdx.x / n3;
  const int node = threadIdx.x % n3;
  const int e = blockIdx.x * EPB + le;
  const bool active = (le < EPB) && (e < D.ne);
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  double* q = sq + le * 7 * n3;
  double* w = sw + le * WORK;
  double pr[7], u0[5];
  if (active) {
    const double* src = V.U + ((size_t)e * n3 + node) * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) u0[v] = src[v];
    prim_point(u0, pr, G);
    if (pr[0] <= 0.0 || pr[4] <= 0.0) atomicOr(&D.status[HDG_STATUS_BAD_PRIM], 1);
    q[0 * n3 + node] = pr[0];
    q[1 * n3 + node] = pr[1];
    q[2 * n3 + node] = pr[2];
    q[3 * n3 + node] = pr[3];
    q[4 * n3 + node] = pr[4];
    q[5 * n3 + node] = pr[6];
    q[6 * n3 + node] = u0[4];
  }
  // flags (VolArgs.mode >> 4; 0 = full RHS): 1 surface integral, 2 Jacobian,
  // 4 accumulate into out (Domain.vol_int), 8 FV residual only, 16 blend + source,
  // 32 indicator only (writes alpha)
  const int vmode = V.mode & 15;
  const int flags = (V.mode >> 4) ? (V.mode >> 4) : (1 | 2 | 16);  // 64: volume from D.vol
  double ut[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if ((flags & 4) && active) {
#pragma unroll
    for (int v = 0; v < 5; ++v) ut[v] = V.out[((size_t)e * n3 + node) * 5 + v];
  }
  if (flags & (8 | 32)) {
    // FV residual only / indicator only: no DG volume term
  } else if (flags & 64) {
    // volume integral precomputed by elem_kernel (Navier-Stokes path)
    if (active) {
#pragma unroll
      for (int v = 0; v < 5; ++v) ut[v] = D.vol[((size_t)e * n3 + node) * 5 + v];
    }
  } else if (SPLIT) {
    // k_vol_int_split (:142-209): per direction, acc_m = sum_alpha Dsplit[m,alpha] F#(m,alpha)
    // in ascending alpha -- the order in which the reference's symmetric pair loop
    // accumulates into acc[m]; F# is bitwise symmetric in its two nodes.
    const double* Ds = sb + DM::oDsplit;
    for (int d = 0; d < 3; ++d) {
      __syncthreads();
      if (active) {
        const double* js = D.Ja + (((size_t)e * 3 + d) * n3 + node) * 3;
        w[0 * n3 + node] = js[0];
        w[1 * n3 + node] = js[1];
        w[2 * n3 + node] = js[2];
        if (VISC) {
          const double* fs = D.Fvis + ((size_t)e * 3 + d) * 4 * n3 + node;
#pragma unroll
          for (int v = 0; v < 4; ++v) w[(3 + v) * n3 + node] = fs[v * n3];
        }
      }
      __syncthreads();
      if (active) {
        const int m = d == 0 ? i : (d == 1 ? j : k);
        const int stride = d == 0 ? 1 : (d == 1 ? n1 : n2);
        const int base = node - m * stride;
        const double rm = pr[0], um = pr[1], vm = pr[2], wm = pr[3], pm = pr[4], hm = pr[6];
        const double jxm = w[0 * n3 + node], jym = w[1 * n3 + node], jzm = w[2 * n3 + node];
        double fvm[4];
        if (VISC) {
#pragma unroll
          for (int v = 0; v < 4; ++v) fvm[v] = w[(3 + v) * n3 + node];
        }
        double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int al = 0; al < n1; ++al) {
          const int na = base + al * stride;
          double fs[5];
          kep_flux(rm, um, vm, wm, pm, hm, q[0 * n3 + na], q[1 * n3 + na], q[2 * n3 + na],
                   q[3 * n3 + na], q[4 * n3 + na], q[5 * n3 + na],
                   0.5 * (jxm + w[0 * n3 + na]), 0.5 * (jym + w[1 * n3 + na]),
                   0.5 * (jzm + w[2 * n3 + na]), fs);
          if (VISC) {
#pragma unroll
            for (int v = 1; v < 5; ++v) fs[v] += 0.5 * (fvm[v - 1] + w[(2 + v) * n3 + na]);
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
    // k_vol_int_standard (:109-139): nodal contravariant fluxes, weak Dhat contraction
    if (active) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double* js = D.Ja + (((size_t)e * 3 + a) * n3 + node) * 3;
        double f[5];
        euler_flux_dir(pr[0], pr[1], pr[2], pr[3], pr[4], u0[4], js[0], js[1], js[2], f);
        if (VISC) {
          const double* fs = D.Fvis + ((size_t)e * 3 + a) * 4 * n3 + node;
#pragma unroll
          for (int v = 1; v < 5; ++v) f[v] += fs[(v - 1) * n3];
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
  // gather surface integral (k_surf_int, :333-358), one writer per DOF, loc 0..5
  if (active && (flags & 1)) {
    const bool lgl = D.node_type == 0;
#pragma unroll
    for (int loc = 0; loc < 6; ++loc) {
      int m, a, b;
      face_coords(loc >> 1, i, j, k, m, a, b);
      if (lgl && m != ((loc & 1) ? N : 0)) continue;
      const int info = D.ef_info[e * 6 + loc];
      const int s = info >> 3, code = info & 3;
      const double sign = ((info >> 2) & 1) ? -1.0 : 1.0;
      const double wt = sign * sb[((loc & 1) ? DM::oLhp : DM::oLhm) + m];
      int p, qq;
      orient<N>(code, a, b, p, qq);
      const double* fs = D.fstar + ((size_t)s * n2 + qq * n1 + p) * 5;
#pragma unroll
      for (int v = 0; v < 5; ++v) ut[v] += wt * fs[v];
    }
  }
  if (active && (flags & 2)) {
    // k_apply_jac: Ut *= -1/J
    const double wj = -D.invJ[(size_t)e * n3 + node];
#pragma unroll
    for (int v = 0; v < 5; ++v) ut[v] *= wj;
  }
  if (SHOCK && (flags & (8 | 16 | 32))) {
    // ---- indicator (src/shock.py:46-110) ----
    __syncthreads();
    double* ind = w;            // [n3]
    double* t1 = w + n3;
    double* t2 = w + 2 * n3;
    if (flags & 8) {
      if (active && node == 0) s_alpha[le] = 1.0;
    } else if (P.indicator == 0) {
      if (active) {
        const double rho = u0[0];
        const double pp = (G.gamma - 1.0) *
                          (u0[4] - 0.5 * (u0[1] * u0[1] + u0[2] * u0[2] + u0[3] * u0[3]) / rho);
        ind[node] = rho * pp;
      }
      __syncthreads();
      const double* Vi = sb + DM::oVinv;
      if (active) {
        double acc = 0.0;
        for (int mm = 0; mm < n1; ++mm) acc += Vi[i * n1 + mm] * ind[k * n2 + j * n1 + mm];
        t1[node] = acc;
      }
      __syncthreads();
      if (active) {
        double acc = 0.0;
        for (int mm = 0; mm < n1; ++mm) acc += Vi[j * n1 + mm] * t1[k * n2 + mm * n1 + i];
        t2[node] = acc;
      }
      __syncthreads();
      if (active) {
        double acc = 0.0;
        for (int mm = 0; mm < n1; ++mm) acc += Vi[k * n1 + mm] * t2[mm * n2 + j * n1 + i];
        t1[node] = acc;
      }
      __syncthreads();
      if (active && node == 0) {
        // sequential sums in (k, j, i) order, as the reference
        double total = 0.0, clip1 = 0.0, clip2 = 0.0;
        for (int nn = 0; nn < n3; ++nn) {
          const int ii = nn % n1, jj = (nn / n1) % n1, kk = nn / n2;
          const double m2 = t1[nn] * t1[nn];
          total += m2;
          if (kk < N && jj < N && ii < N) clip1 += m2;
          if (kk < N - 1 && jj < N - 1 && ii < N - 1) clip2 += m2;
        }
        double energy = 0.0;
        if (total > 1e-300) energy = (total - clip1) / total;
        if (clip1 > 1e-300) {
          const double e2 = (clip1 - clip2) / clip1;
          if (e2 > energy) energy = e2;
        }
        double a = 1.0 / (1.0 + exp(P.ind_slope * (energy - P.ind_threshold)));
        if (a > P.alpha_max) a = P.alpha_max;
        if (a < P.alpha_min) a = 0.0;
        s_alpha[le] = a;
      }
    } else {
      if (active && node == 0) s_alpha[le] = dmin(P.alpha_const, P.alpha_max);
    }
    __syncthreads();
    const double alpha = (le < EPB) ? s_alpha[le] : 0.0;
    if (active && node == 0 && !(flags & 8)) D.alpha[e] = alpha;
    // ---- FV subcell residual + blend (src/shock.py:113-210), flagged elements only ----
    if (flags & 32) return;   // indicator only (shock.indicator_alpha)
    double rfv[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    bool any = false;
    for (int l2 = 0; l2 < EPB; ++l2) any |= s_alpha[l2] > 0.0;
    if (any) {
      double* Fl = w;   // [n2][n1+1][5] interface fluxes of one direction
      const double* fvms[3] = {D.fvm0, D.fvm1, D.fvm2};
      for (int d = 0; d < 3; ++d) {
        __syncthreads();
        if (active && alpha > 0.0) {
          const int loc_m = 2 * d, loc_p = 2 * d + 1;
          const int inm = D.ef_info[e * 6 + loc_m], inp = D.ef_info[e * 6 + loc_p];
          for (int t = node; t < n2 * (n1 + 1); t += n3) {
            const int line = t / (n1 + 1), h = t % (n1 + 1);
            const int a = line % n1, b = line / n1;     // tangential (a, b) of loc 2d
            double f[5];
            if (h == 0 || h == n1) {
              const int info = h == 0 ? inm : inp;
              const double sg = ((info >> 2) & 1) ? -1.0 : 1.0;
              int p, qq;
              orient<N>(info & 3, a, b, p, qq);
              const double* fs = D.fstar + ((size_t)(info >> 3) * n2 + qq * n1 + p) * 5;
              const double fac = h == 0 ? -sg : sg;
#pragma unroll
              for (int v = 0; v < 5; ++v) f[v] = fac * fs[v];
            } else {
              const int nL = vol_node<N>(loc_m, a, b, h - 1), nR = vol_node<N>(loc_m, a, b, h);
              // fvm layouts: d=0 [e,b,a,h]; d=1 [e,a,b,h]; d=2 [e,b,a,h]
              const int r1 = d == 1 ? a : b, r2 = d == 1 ? b : a;
              const double* mv = fvms[d] + ((((size_t)e * n1 + r1) * n1 + r2) * (n1 + 1) + h) * 3;
              const double mx = mv[0], my = mv[1], mz = mv[2];
              const double sn = sqrt(mx * mx + my * my + mz * mz);
              const double L[5] = {q[0 * n3 + nL], q[1 * n3 + nL], q[2 * n3 + nL], q[3 * n3 + nL],
                                   q[4 * n3 + nL]};
              const double R[5] = {q[0 * n3 + nR], q[1 * n3 + nR], q[2 * n3 + nR], q[3 * n3 + nR],
                                   q[4 * n3 + nR]};
              riemann(P.fv_solver, L, q[6 * n3 + nL], R, q[6 * n3 + nR], mx / sn, my / sn, mz / sn,
                      G.gamma, f);
#pragma unroll
              for (int v = 0; v < 5; ++v) f[v] = f[v] * sn;
            }
            double* o = Fl + (line * (n1 + 1) + h) * 5;
#pragma unroll
            for (int v = 0; v < 5; ++v) o[v] = f[v];
          }
        }
        __syncthreads();
        if (active && alpha > 0.0) {
          int m, a, b;
          face_coords(d, i, j, k, m, a, b);
          const double iwh = sb[DM::oIW + m];
          const double* F0 = Fl + ((b * n1 + a) * (n1 + 1) + m) * 5;
#pragma unroll
          for (int v = 0; v < 5; ++v) rfv[v] -= (F0[5 + v] - F0[v]) * iwh;
        }
      }
      if (active && alpha > 0.0) {
        const double iw = D.invJ[(size_t)e * n3 + node];
        const double bb = 1.0 - alpha;
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          rfv[v] *= iw;
          ut[v] = (flags & 8) ? rfv[v] : bb * ut[v] + alpha * rfv[v];
        }
      }
    }
  }
  if (!active) return;
  const double tstage = V.time ? V.time[0] + V.c * V.time[1] : V.t_host;
  if (P.source && (flags & 16)) add_mms_source(P, D.x + ((size_t)e * n3 + node) * 3, tstage, ut);
  const size_t o = ((size_t)e * n3 + node) * 5;
  if (vmode == HDG_MODE_STORE_UT) {
#pragma unroll
    for (int v = 0; v < 5; ++v) V.out[o + v] = ut[v];
  } else {
    // rk_step (src/timedisc.py:132-137) without FMA contraction
    const double dt = V.time[1];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const double du = vmode == HDG_MODE_LSERK_FIRST
                            ? __dmul_rn(dt, ut[v])
                            : __dadd_rn(__dmul_rn(V.out[o + v], V.A), __dmul_rn(dt, ut[v]));
      V.out[o + v] = du;
      V.U[o + v] = __dadd_rn(u0[v], __dmul_rn(V.B, du));
    }
  }
}

// ---------------------------------------------------------------------------
// TGV analysis partial sums (k_analysis_partials, src/testcases.py:190-226): one
// thread per element, its nodes in (k, j, i) order and the reference's operation
// order, so each element row is independent of the rank layout. out[e][9] =
// mass, 3 momenta, energy, rho u.u, mu/mu0 |curl u|^2, mu/mu0 (div u)^2, volume.
// g may be null for Euler (rows 6 and 7 stay 0).
template <int N>
__global__ void __launch_bounds__(128) analysis_kernel(hdg_domain D, hdg_params P,
                                                       const double* __restrict__ U,
                                                       const double* __restrict__ g, double mu0,
                                                       double* __restrict__ out) {
  constexpr int n1 = N + 1, n2 = n1 * n1, n3 = n2 * n1;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= D.ne) return;
  const Gas G = make_gas(P);
  const double* w = D.basis + Dim<N>::oW;
  double acc[9] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int node = 0; node < n3; ++node) {
    const int i = node % n1, j = (node / n1) % n1, k = node / n2;
    const size_t t = (size_t)e * n3 + node;
    const double dv = D.J[t] * w[i] * w[j] * w[k];
    const double* u = U + t * 5;
    const double rho = u[0], mx = u[1], my = u[2], mz = u[3];
    acc[0] += dv * rho;
    acc[1] += dv * mx;
    acc[2] += dv * my;
    acc[3] += dv * mz;
    acc[4] += dv * u[4];
    acc[5] += dv * (mx * mx + my * my + mz * mz) / rho;
    if (P.viscous) {
      const double p = (G.gamma - 1.0) * (u[4] - 0.5 * (mx * mx + my * my + mz * mz) / rho);
      const double T = p / (rho * G.R);
      const double mu = viscosity(T, G) / mu0;
      const double* gg = g + t * 12;   // [d][l], d = d/dx,y,z, l = u,v,w,T
      const double wx = gg[1 * 4 + 2] - gg[2 * 4 + 1];
      const double wy = gg[2 * 4 + 0] - gg[0 * 4 + 2];
      const double wz = gg[0 * 4 + 1] - gg[1 * 4 + 0];
      const double div = gg[0 * 4 + 0] + gg[1 * 4 + 1] + gg[2 * 4 + 2];
      acc[6] += dv * mu * (wx * wx + wy * wy + wz * wz);
      acc[7] += dv * mu * div * div;
    }
    acc[8] += dv;
  }
#pragma unroll
  for (int v = 0; v < 9; ++v) out[(size_t)e * 9 + v] = acc[v];
}

// ---------------------------------------------------------------------------
// k_local_dt of one node (src/operator.py:460-487) from its conserved state, the
// reference's operations in order; +inf when no bound applies
template <int N>
__device__ __forceinline__ double node_dt(const double u[5], const hdg_domain& D,
                                          const hdg_params& P, const Gas& G, long e, long node,
                                          double J, double cfl, double cfl_visc) {
  constexpr int n3 = (N + 1) * (N + 1) * (N + 1);
  double best = __longlong_as_double(0x7ff0000000000000LL);
  double pr[7];
  prim_point(u, pr, G);
  const double a = sqrt(G.gamma * pr[4] / pr[0]);
  const double scale = 2.0 * N + 1.0;
  double lam = 0.0, metric2 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double* js = D.Ja + ((e * 3 + d) * n3 + node) * 3;
    const double jx = js[0], jy = js[1], jz = js[2];
    const double nrm = sqrt(jx * jx + jy * jy + jz * jz);
    const double vn = pr[1] * jx + pr[2] * jy + pr[3] * jz;
    lam += fabs(vn) + a * nrm;
    metric2 += nrm * nrm;
  }
  const double dta = cfl * 2.0 * J / (scale * lam);
  if (dta < best) best = dta;
  if (P.viscous) {
    const double mu = viscosity(pr[5], G);
    const double nu = mu / pr[0] * dmax(4.0 / 3.0, G.gamma / G.Pr);
    if (nu > 0.0) {
      const double tj = 2.0 * J;
      const double dtv = cfl_visc * (tj * tj) / (scale * scale * metric2 * nu);
      if (dtv < best) best = dtv;
    }
  }
  return best;
}

// block-wide min of the dt bit patterns (exact: positive doubles order like their
// bits) and OR of the non-finite flags, one atomic each per block
__device__ __forceinline__ void reduce_dt_block(const hdg_domain& D, unsigned long long bits,
                                                int nonfinite) {
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, bits, off);
    bits = o < bits ? o : bits;
    nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, off);
  }
  __shared__ unsigned long long sbits[32];
  __shared__ int snf[32];
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sbits[wid] = bits;
    snf[wid] = nonfinite;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      bits = sbits[w] < bits ? sbits[w] : bits;
      nonfinite |= snf[w];
    }
    atomicMin(reinterpret_cast<unsigned long long*>(D.dt_bits), bits);
    if (nonfinite) atomicOr(&D.status[HDG_STATUS_NONFINITE], 1);
  }
}

// k_local_dt + isfinite(U): grid-stride over nodes, one atomic min per block
template <int N>
__global__ void __launch_bounds__(256) dt_kernel(hdg_domain D, hdg_params P,
                                                 const double* __restrict__ U, double cfl,
                                                 double cfl_visc) {
  constexpr int n3 = (N + 1) * (N + 1) * (N + 1);
  const Gas G = make_gas(P);
  unsigned long long bits = 0x7ff0000000000000ULL;   // +inf
  int nonfinite = 0;
  const long total = (long)D.ne * n3;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    double u[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      u[v] = U[t * 5 + v];
      nonfinite |= !isfinite(u[v]);
    }
    const double best = node_dt<N>(u, D, P, G, t / n3, t % n3, D.J[t], cfl, cfl_visc);
    if (best >= 0.0) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(best);
      bits = b < bits ? b : bits;
    }
  }
  reduce_dt_block(D, bits, nonfinite);
}

// k_cons_to_prim (:76-86)
__global__ void cons_to_prim_kernel(hdg_domain D, hdg_params P, const double* __restrict__ U,
                                    double* __restrict__ prim, long n) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const Gas G = make_gas(P);
  double u[5], pr[7];
  for (int v = 0; v < 5; ++v) u[v] = U[t * 5 + v];
  prim_point(u, pr, G);
  if (pr[0] <= 0.0 || pr[4] <= 0.0) atomicOr(&D.status[HDG_STATUS_BAD_PRIM], 1);
  for (int v = 0; v < 7; ++v) prim[t * 7 + v] = pr[v];
}

// raw k_surf_int (:333-358) and k_apply_jac (:361-370), API granularity
template <int N>
__global__ void surf_int_kernel(hdg_domain D, const double* __restrict__ fstar,
                                double* __restrict__ Ut) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)D.ne * n3) return;
  const int e = (int)(t / n3), node = (int)(t % n3);
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  double ut[5];
  for (int v = 0; v < 5; ++v) ut[v] = Ut[t * 5 + v];
  for (int loc = 0; loc < 6; ++loc) {
    int m, a, b;
    face_coords(loc >> 1, i, j, k, m, a, b);
    const int info = D.ef_info[e * 6 + loc];
    const int s = info >> 3, code = info & 3;
    const double sign = ((info >> 2) & 1) ? -1.0 : 1.0;
    const double wt = sign * D.basis[((loc & 1) ? DM::oLhp : DM::oLhm) + m];
    int p, q;
    orient<N>(code, a, b, p, q);
    const double* fs = fstar + ((size_t)s * n2 + q * n1 + p) * 5;
    for (int v = 0; v < 5; ++v) ut[v] += wt * fs[v];
  }
  for (int v = 0; v < 5; ++v) Ut[t * 5 + v] = ut[v];
}

__global__ void apply_jac_kernel(const double* __restrict__ J, double* __restrict__ Ut, long n) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double w = -1.0 / J[t];
  for (int v = 0; v < 5; ++v) Ut[t * 5 + v] *= w;
}

// pack the rank's own face traces of partition-boundary sides, in the a-priori
// neighbour order (_pack_sides, src/parallel.py:348-358): buf[k][q][p][5]
template <int N, bool LGL>
__global__ void pack_traces_kernel(hdg_domain D, const double* __restrict__ U,
                                   const int32_t* __restrict__ sides, int n, double* __restrict__ buf) {
  constexpr int n2 = (N + 1) * (N + 1);
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)n * n2) return;
  const int kk = (int)(t / n2), fq = (int)(t % n2);
  const int s = sides[kk];
  const int role = reinterpret_cast<const int4*>(D.side_info)[s].x >= 0 ? 0 : 1;
  double u[5];
  load_trace<N, LGL>(D, U, s, role, fq / (N + 1), fq % (N + 1), u);
#pragma unroll
  for (int v = 0; v < 5; ++v) buf[t * 5 + v] = u[v];
}

// ---------------------------------------------------------------------------
// Partition-boundary exchange over NVLink peer memory (one node): the pack is
// fused with the remote store -- each row goes straight into the neighbour's
// array (its UL/UR halo row, fvface row or f* row, mapped by CUDA IPC) -- and
// the last block to finish publishes the phase epoch to every neighbour's flag
// word. No staging buffers, no unpack, no communication kernels on the SMs.
template <int N>
__global__ void __launch_bounds__(256) peer_send_traces_kernel(
    hdg_domain D, const double* __restrict__ U, const int32_t* __restrict__ nbr,
    const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int n,
    const unsigned long long* __restrict__ dst_base, const unsigned long long* __restrict__ flag_ptrs,
    int n_nbr, unsigned* counter, unsigned long long* epoch) {
  constexpr int n2 = (N + 1) * (N + 1);
  // grid-stride (few blocks: each pays one system fence + counter atomic at the end)
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < (long)n * n2;
       t += (long)gridDim.x * blockDim.x) {
    const int kk = (int)(t / n2), fq = (int)(t % n2);
    const int s = src[kk];
    const int role = reinterpret_cast<const int4*>(D.side_info)[s].x >= 0 ? 0 : 1;   // own trace
    double u[5];
    load_trace<N, true>(D, U, s, role, fq / (N + 1), fq % (N + 1), u);
    double* out = reinterpret_cast<double*>(dst_base[nbr[kk]]) + ((size_t)dst[kk] * n2 + fq) * 5;
#pragma unroll
    for (int v = 0; v < 5; ++v) out[v] = u[v];
  }
  publish_epoch(counter, flag_ptrs, n_nbr, epoch);
}
