// API-granularity kernels of the reference's Python surface that are not on the
// production stage path (included in both kernel sets after elem2.cuh): the point
// physics of hexdg.equations evaluated for a batch of independent inputs, the
// manufactured-solution source at arbitrary points, and the three split lifting
// calls Domain.lift_fill / lift_volume / lift_finish. Same arithmetic, same order
// as the reference routines they cite.

enum {
  HDG_POINT_EULER_FLUX_DIR = 0,   // pt_euler_flux_dir   (src/equations.py:93-102)
  HDG_POINT_VISCOUS_FLUX_DIR = 1, // pt_viscous_flux_dir (:262-285), mu/lam from T
  HDG_POINT_RIEMANN = 2,          // pt_riemann          (:219-232)
  HDG_POINT_SPLIT_KEP = 3,        // pt_split_flux_kep   (:235-259)
  HDG_POINT_VISCOSITY = 4,        // pt_viscosity        (:75-80)
  HDG_POINT_CONDUCTIVITY = 5,     // pt_conductivity     (:83-85)
};

__host__ __device__ constexpr int point_width_in(int op) {
  return op == 0 ? 9 : op == 1 ? 19 : op == 2 ? 15 : op == 3 ? 15 : 1;
}
__host__ __device__ constexpr int point_width_out(int op) { return op >= 4 ? 1 : 5; }

__global__ void point_kernel(hdg_params P, int op, int solver, int n,
                             const double* __restrict__ in, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const Gas G = make_gas(P);
  const double* x = in + (size_t)t * point_width_in(op);
  double* o = out + (size_t)t * point_width_out(op);
  double f[5];
  switch (op) {
    case HDG_POINT_EULER_FLUX_DIR:
      euler_flux_dir(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], x[8], f);
      break;
    case HDG_POINT_VISCOUS_FLUX_DIR: {
      const double mu = viscosity(x[3], G);
      const double lam = conductivity(mu, G);
      viscous_flux_dir(x[0], x[1], x[2], mu, lam, x + 4, x[16], x[17], x[18], f);
      break;
    }
    case HDG_POINT_RIEMANN:
      riemann(solver, x, x[5], x + 6, x[11], x[12], x[13], x[14], G.gamma, f);
      break;
    case HDG_POINT_SPLIT_KEP:
      kep_flux(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], x[8], x[9], x[10], x[11], x[12],
               x[13], x[14], f);
      break;
    case HDG_POINT_VISCOSITY:
      o[0] = viscosity(x[0], G);
      return;
    default:
      o[0] = conductivity(x[0], G);
      return;
  }
#pragma unroll
  for (int v = 0; v < 5; ++v) o[v] = f[v];
}

int run_point(const hdg_params& P, int op, int solver, int n, const double* in, double* out,
              cudaStream_t st) {
  if (n <= 0) return 0;
  if (op < 0 || op > 5) {
    hdg::set_error("hdg_point_eval: unknown op %d", op);
    return -1;
  }
  point_kernel<<<(n + 127) / 128, 128, 0, st>>>(P, op, solver, n, in, out);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    hdg::set_error("point_kernel launch failed: %s", cudaGetErrorString(err));
    return -4;
  }
  hdg::count_launch();
  return 0;
}

// testcases.mms_source / k_mms_source (src/testcases.py:51-70) at n points
__global__ void mms_points_kernel(hdg_params P, int n, const double* __restrict__ x, double t,
                                  double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ut[5];
  for (int v = 0; v < 5; ++v) ut[v] = out[(size_t)i * 5 + v];
  add_mms_source(P, x + (size_t)i * 3, t, ut);
  for (int v = 0; v < 5; ++v) out[(size_t)i * 5 + v] = ut[v];
}

int run_mms_points(const hdg_params& P, int n, const double* x, double t, double* out,
                   cudaStream_t st) {
  if (n <= 0) return 0;
  mms_points_kernel<<<(n + 127) / 128, 128, 0, st>>>(P, n, x, t, out);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    hdg::set_error("mms_points_kernel launch failed: %s", cudaGetErrorString(err));
    return -4;
  }
  hdg::count_launch();
  return 0;
}

// Domain.lift_fill -> k_lift_fill (src/operator.py:377-391): vstar on the listed
// sides from the UL / UR trace arrays, one thread per (side, q, p)
template <int N>
__global__ void lift_fill_kernel(hdg_domain D, hdg_params P, const int32_t* __restrict__ sides,
                                 int nsides) {
  constexpr int n1 = N + 1, n2 = n1 * n1;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)nsides * n2) return;
  const int s = sides[t / n2], fq = (int)(t % n2);
  const Gas G = make_gas(P);
  const size_t o = (size_t)s * n2 + fq;
  double pl[7], pr[7];
  prim_point(D.UL + o * 5, pl, G);
  prim_point(D.UR + o * 5, pr, G);
  double* vs = D.vstar + o * 4;
  vs[0] = 0.5 * (pl[1] + pr[1]);
  vs[1] = 0.5 * (pl[2] + pr[2]);
  vs[2] = 0.5 * (pl[3] + pr[3]);
  vs[3] = 0.5 * (pl[5] + pr[5]);
}

// Domain.lift_volume -> k_lift_volume (:394-418): g = the weak volume term from the
// prims of U (no surface term, no 1/J), one thread per node
template <int N>
__global__ void lift_volume_kernel(hdg_domain D, hdg_params P, const double* __restrict__ U) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)D.ne * n3) return;
  const int e = (int)(t / n3), node = (int)(t % n3);
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  const Gas G = make_gas(P);
  const double* Dh = D.basis + DM::oDhat;
  const double* Ja = D.Ja + (size_t)e * 3 * n3 * 3;
  const double* Ue = U + (size_t)e * n3 * 5;
  double g[12];
  for (int c = 0; c < 12; ++c) g[c] = 0.0;
  for (int al = 0; al < n1; ++al) {
    const double di = Dh[i * n1 + al], dj = Dh[j * n1 + al], dk = Dh[k * n1 + al];
    const int ni = k * n2 + j * n1 + al, nj = k * n2 + al * n1 + i, nk = al * n2 + j * n1 + i;
    double pi[7], pj[7], pk[7];
    prim_point(Ue + ni * 5, pi, G);
    prim_point(Ue + nj * 5, pj, G);
    prim_point(Ue + nk * 5, pk, G);
    for (int d = 0; d < 3; ++d) {
      const double jai = di * Ja[(0 * n3 + ni) * 3 + d];
      const double jaj = dj * Ja[(1 * n3 + nj) * 3 + d];
      const double jak = dk * Ja[(2 * n3 + nk) * 3 + d];
      for (int l = 0; l < 4; ++l) {
        const int lp = l < 3 ? 1 + l : 5;   // velocities, then temperature
        g[d * 4 + l] += jai * pi[lp] + jaj * pj[lp] + jak * pk[lp];
      }
    }
  }
  double* dg = D.g + ((size_t)e * n3 + node) * 12;
  for (int c = 0; c < 12; ++c) dg[c] = g[c];
}

// Domain.lift_finish -> k_lift_surf_and_jac (:421-453) + k_viscous_contravariant
// (:89-102): g += surface term from vstar, g *= 1/J, Fvis[e][a][v][node]
template <int N>
__global__ void lift_finish_kernel(hdg_domain D, hdg_params P, const double* __restrict__ U) {
  using DM = Dim<N>;
  constexpr int n1 = DM::n1, n2 = DM::n2, n3 = DM::n3;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)D.ne * n3) return;
  const int e = (int)(t / n3), node = (int)(t % n3);
  const int i = node % n1, j = (node / n1) % n1, k = node / n2;
  const Gas G = make_gas(P);
  double g[12];
  double* dg = D.g + ((size_t)e * n3 + node) * 12;
  for (int c = 0; c < 12; ++c) g[c] = dg[c];
  for (int loc = 0; loc < 6; ++loc) {
    int m, a, b;
    face_coords(loc >> 1, i, j, k, m, a, b);
    const int info = D.ef_info[(size_t)e * 6 + loc];
    const int s = info >> 3;
    const double sign = ((info >> 2) & 1) ? -1.0 : 1.0;
    int p, q;
    orient<N>(info & 3, a, b, p, q);
    const double lh = D.basis[((loc & 1) ? DM::oLhp : DM::oLhm) + m];
    const size_t fo = (size_t)s * n2 + q * n1 + p;
    const double w = sign * lh * D.ssurf[fo];
    for (int dd = 0; dd < 3; ++dd) {
      const double nd = w * D.nvec[fo * 3 + dd];
      for (int l = 0; l < 4; ++l) g[dd * 4 + l] += nd * D.vstar[fo * 4 + l];
    }
  }
  const double iw = 1.0 / D.J[(size_t)e * n3 + node];
  for (int c = 0; c < 12; ++c) {
    g[c] *= iw;
    dg[c] = g[c];
  }
  if (D.Fvis) {
    double pr[7];
    prim_point(U + ((size_t)e * n3 + node) * 5, pr, G);
    const double mu = viscosity(pr[5], G);
    const double lam = conductivity(mu, G);
    for (int a = 0; a < 3; ++a) {
      const double* ja = D.Ja + (((size_t)e * 3 + a) * n3 + node) * 3;
      double fv[5];
      viscous_flux_dir(pr[1], pr[2], pr[3], mu, lam, g, ja[0], ja[1], ja[2], fv);
      for (int v = 0; v < 4; ++v) D.Fvis[(((size_t)e * 3 + a) * 4 + v) * n3 + node] = fv[v + 1];
    }
  }
}

template <int N>
static int lift_split_n(const hdg_domain& D, const hdg_params& P, int which, const double* U,
                        const int32_t* sides, int nsides, cudaStream_t st) {
  constexpr int n2 = (N + 1) * (N + 1), n3 = n2 * (N + 1);
  if (which == 0) {
    if (nsides <= 0) return 0;
    lift_fill_kernel<N><<<(int)(((long)nsides * n2 + 127) / 128), 128, 0, st>>>(D, P, sides, nsides);
  } else {
    const long tot = (long)D.ne * n3;
    if (tot == 0) return 0;
    if (which == 1)
      lift_volume_kernel<N><<<(int)((tot + 127) / 128), 128, 0, st>>>(D, P, U);
    else
      lift_finish_kernel<N><<<(int)((tot + 127) / 128), 128, 0, st>>>(D, P, U);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    hdg::set_error("lifting API kernel launch failed: %s", cudaGetErrorString(err));
    return -4;
  }
  hdg::count_launch();
  return 0;
}

int run_lift_split(const hdg_domain& D, const hdg_params& P, int which, const double* U,
                   const int32_t* sides, int nsides, cudaStream_t st) {
  switch (D.N) {
    case 1: return lift_split_n<1>(D, P, which, U, sides, nsides, st);
    case 2: return lift_split_n<2>(D, P, which, U, sides, nsides, st);
    case 3: return lift_split_n<3>(D, P, which, U, sides, nsides, st);
    case 4: return lift_split_n<4>(D, P, which, U, sides, nsides, st);
    case 5: return lift_split_n<5>(D, P, which, U, sides, nsides, st);
    case 6: return lift_split_n<6>(D, P, which, U, sides, nsides, st);
    case 7: return lift_split_n<7>(D, P, which, U, sides, nsides, st);
    default: hdg::set_error("unsupported degree N=%d (1..7)", (int)D.N); return -2;
  }
}
