/*
 * ORACLE -- test infrastructure only. CPU restatement of the reference's
 * numba kernels (hexdg, /root/reference/pkg/src/hexdg/{operator,equations,
 * shock,testcases}.py), used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg as the CHECKER and the CPU baseline.
 * Never linked into or called by the product path.
 *
 * Every function cites the reference kernel it restates and performs the same
 * IEEE float64 operations in the same order (compiled with -ffp-contract=off,
 * no -ffast-math): results are bit-identical to the reference's numba kernels
 * (pinned against golden vectors produced by the reference itself,
 * tests/golden/make_golden.py). OpenMP parallelises only loops whose
 * iterations are independent (as the reference's prange loops).
 *
 * Layouts are the reference's: U[e][k][j][i][5], Ja[e][a][k][j][i][c],
 * faces [s][q][p][v], g[e][k][j][i][d][l], Fvis[e][k][j][i][a][v],
 * fvm_d[e][r1][r2][h][3]; index arrays are int64, ef_sign float64.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

typedef int64_t i64;

#define NVAR 5
#define NPRIM 7
#define NLIFT 4

static inline double pmax(double a, double b) { return (b > a) ? b : a; }  /* python max */
static inline double pmin(double a, double b) { return (b < a) ? b : a; }  /* python min */

/* _prim_point, src/operator.py:55-69 */
static inline void prim_point(const double* U, double* o, double gamma, double R) {
  double rho = U[0];
  double ir = 1.0 / rho;
  double u = U[1] * ir, v = U[2] * ir, w = U[3] * ir;
  double p = (gamma - 1.0) * (U[4] - 0.5 * rho * (u * u + v * v + w * w));
  o[0] = rho; o[1] = u; o[2] = v; o[3] = w; o[4] = p;
  o[5] = p * ir / R;
  o[6] = (U[4] + p) * ir;
}

/* src/equations.py:75-90 */
static inline double pt_viscosity(double T, double mu_ref, double T_ref, int law) {
  if (law == 0) return mu_ref;
  double tr = T / T_ref;
  return mu_ref * 1.4042 * tr * sqrt(tr) / (tr + 0.4042);
}
static inline double pt_conductivity(double mu, double gamma, double R, double Pr) {
  return gamma * R / (gamma - 1.0) * mu / Pr;
}
static inline double pt_sound_speed(double rho, double p, double gamma) { return sqrt(gamma * p / rho); }

/* src/equations.py:93-102 */
static inline void pt_euler_flux_dir(double rho, double u, double v, double w, double p, double rhoE,
                                     double nx, double ny, double nz, double* out) {
  double vn = u * nx + v * ny + w * nz;
  double m = rho * vn;
  out[0] = m;
  out[1] = m * u + p * nx;
  out[2] = m * v + p * ny;
  out[3] = m * w + p * nz;
  out[4] = vn * (rhoE + p);
}

/* src/equations.py:105-121 */
static void pt_llf(double rhoL, double uL, double vL, double wL, double pL, double rhoEL,
                   double rhoR, double uR, double vR, double wR, double pR, double rhoER,
                   double nx, double ny, double nz, double gamma, double* out) {
  double fR[5];
  pt_euler_flux_dir(rhoL, uL, vL, wL, pL, rhoEL, nx, ny, nz, out);
  pt_euler_flux_dir(rhoR, uR, vR, wR, pR, rhoER, nx, ny, nz, fR);
  double vnL = uL * nx + vL * ny + wL * nz;
  double vnR = uR * nx + vR * ny + wR * nz;
  double lam = pmax(fabs(vnL) + pt_sound_speed(rhoL, pL, gamma), fabs(vnR) + pt_sound_speed(rhoR, pR, gamma));
  out[0] = 0.5 * (out[0] + fR[0]) - 0.5 * lam * (rhoR - rhoL);
  out[1] = 0.5 * (out[1] + fR[1]) - 0.5 * lam * (rhoR * uR - rhoL * uL);
  out[2] = 0.5 * (out[2] + fR[2]) - 0.5 * lam * (rhoR * vR - rhoL * vL);
  out[3] = 0.5 * (out[3] + fR[3]) - 0.5 * lam * (rhoR * wR - rhoL * wL);
  out[4] = 0.5 * (out[4] + fR[4]) - 0.5 * lam * (rhoER - rhoEL);
}

/* src/equations.py:124-185 */
static void pt_hllc(double rhoL, double uL, double vL, double wL, double pL, double rhoEL,
                    double rhoR, double uR, double vR, double wR, double pR, double rhoER,
                    double nx, double ny, double nz, double gamma, double* out) {
  double vnL = uL * nx + vL * ny + wL * nz;
  double vnR = uR * nx + vR * ny + wR * nz;
  double aL = pt_sound_speed(rhoL, pL, gamma);
  double aR = pt_sound_speed(rhoR, pR, gamma);
  double sqL = sqrt(rhoL), sqR = sqrt(rhoR);
  double fac = 1.0 / (sqL + sqR);
  double vnRoe = (sqL * vnL + sqR * vnR) * fac;
  double HL = (rhoEL + pL) / rhoL;
  double HR = (rhoER + pR) / rhoR;
  double HRoe = (sqL * HL + sqR * HR) * fac;
  double u2Roe = ((sqL * (uL * uL + vL * vL + wL * wL) + sqR * (uR * uR + vR * vR + wR * wR)) * fac);
  double aRoe = sqrt(pmax((gamma - 1.0) * (HRoe - 0.5 * u2Roe), 1e-300));
  double sL = pmin(vnL - aL, vnRoe - aRoe);
  double sR = pmax(vnR + aR, vnRoe + aRoe);
  if (sL >= 0.0) { pt_euler_flux_dir(rhoL, uL, vL, wL, pL, rhoEL, nx, ny, nz, out); return; }
  if (sR <= 0.0) { pt_euler_flux_dir(rhoR, uR, vR, wR, pR, rhoER, nx, ny, nz, out); return; }
  double sM = (pR - pL + rhoL * vnL * (sL - vnL) - rhoR * vnR * (sR - vnR)) /
              (rhoL * (sL - vnL) - rhoR * (sR - vnR));
  double us[5];
  if (sM >= 0.0) {
    pt_euler_flux_dir(rhoL, uL, vL, wL, pL, rhoEL, nx, ny, nz, out);
    double rho_s = rhoL * (sL - vnL) / (sL - sM);
    us[0] = rho_s;
    us[1] = rho_s * (uL + (sM - vnL) * nx);
    us[2] = rho_s * (vL + (sM - vnL) * ny);
    us[3] = rho_s * (wL + (sM - vnL) * nz);
    us[4] = rho_s * (rhoEL / rhoL + (sM - vnL) * (sM + pL / (rhoL * (sL - vnL))));
    out[0] += sL * (us[0] - rhoL);
    out[1] += sL * (us[1] - rhoL * uL);
    out[2] += sL * (us[2] - rhoL * vL);
    out[3] += sL * (us[3] - rhoL * wL);
    out[4] += sL * (us[4] - rhoEL);
  } else {
    pt_euler_flux_dir(rhoR, uR, vR, wR, pR, rhoER, nx, ny, nz, out);
    double rho_s = rhoR * (sR - vnR) / (sR - sM);
    us[0] = rho_s;
    us[1] = rho_s * (uR + (sM - vnR) * nx);
    us[2] = rho_s * (vR + (sM - vnR) * ny);
    us[3] = rho_s * (wR + (sM - vnR) * nz);
    us[4] = rho_s * (rhoER / rhoR + (sM - vnR) * (sM + pR / (rhoR * (sR - vnR))));
    out[0] += sR * (us[0] - rhoR);
    out[1] += sR * (us[1] - rhoR * uR);
    out[2] += sR * (us[2] - rhoR * vR);
    out[3] += sR * (us[3] - rhoR * wR);
    out[4] += sR * (us[4] - rhoER);
  }
}

/* src/equations.py:235-259 */
static inline void pt_split_flux_kep(double rhoL, double uL, double vL, double wL, double pL, double hL,
                                     double rhoR, double uR, double vR, double wR, double pR, double hR,
                                     double jx, double jy, double jz, double* out) {
  double rm = 0.5 * (rhoL + rhoR);
  double um = 0.5 * (uL + uR);
  double vm = 0.5 * (vL + vR);
  double wm = 0.5 * (wL + wR);
  double pm = 0.5 * (pL + pR);
  double hm = 0.5 * (hL + hR);
  double vn = um * jx + vm * jy + wm * jz;
  double m = rm * vn;
  out[0] = m;
  out[1] = m * um + pm * jx;
  out[2] = m * vm + pm * jy;
  out[3] = m * wm + pm * jz;
  out[4] = m * hm;
}

/* src/equations.py:188-210 */
static void pt_llf_split(double rhoL, double uL, double vL, double wL, double pL, double rhoEL,
                         double rhoR, double uR, double vR, double wR, double pR, double rhoER,
                         double nx, double ny, double nz, double gamma, double* out) {
  pt_split_flux_kep(rhoL, uL, vL, wL, pL, (rhoEL + pL) / rhoL, rhoR, uR, vR, wR, pR,
                    (rhoER + pR) / rhoR, nx, ny, nz, out);
  double vnL = uL * nx + vL * ny + wL * nz;
  double vnR = uR * nx + vR * ny + wR * nz;
  double lam = pmax(fabs(vnL) + pt_sound_speed(rhoL, pL, gamma), fabs(vnR) + pt_sound_speed(rhoR, pR, gamma));
  out[0] -= 0.5 * lam * (rhoR - rhoL);
  out[1] -= 0.5 * lam * (rhoR * uR - rhoL * uL);
  out[2] -= 0.5 * lam * (rhoR * vR - rhoL * vL);
  out[3] -= 0.5 * lam * (rhoR * wR - rhoL * wL);
  out[4] -= 0.5 * lam * (rhoER - rhoEL);
}

/* src/equations.py:219-232 */
static void pt_riemann(int solver, const double* pl, double rhoEL, const double* pr, double rhoER,
                       double nx, double ny, double nz, double gamma, double* out) {
  if (solver == 1)
    pt_hllc(pl[0], pl[1], pl[2], pl[3], pl[4], rhoEL, pr[0], pr[1], pr[2], pr[3], pr[4], rhoER, nx, ny, nz, gamma, out);
  else if (solver == 2)
    pt_llf_split(pl[0], pl[1], pl[2], pl[3], pl[4], rhoEL, pr[0], pr[1], pr[2], pr[3], pr[4], rhoER, nx, ny, nz, gamma, out);
  else
    pt_llf(pl[0], pl[1], pl[2], pl[3], pl[4], rhoEL, pr[0], pr[1], pr[2], pr[3], pr[4], rhoER, nx, ny, nz, gamma, out);
}

/* src/equations.py:262-285; g[d*4 + l] */
static void pt_viscous_flux_dir(double u, double v, double w, double mu, double lam, const double* g,
                                double nx, double ny, double nz, double* out) {
  double dudx = g[0], dvdx = g[1], dwdx = g[2], dTdx = g[3];
  double dudy = g[4], dvdy = g[5], dwdy = g[6], dTdy = g[7];
  double dudz = g[8], dvdz = g[9], dwdz = g[10], dTdz = g[11];
  double divu = dudx + dvdy + dwdz;
  double txx = mu * (2.0 * dudx - 2.0 / 3.0 * divu);
  double tyy = mu * (2.0 * dvdy - 2.0 / 3.0 * divu);
  double tzz = mu * (2.0 * dwdz - 2.0 / 3.0 * divu);
  double txy = mu * (dudy + dvdx);
  double txz = mu * (dudz + dwdx);
  double tyz = mu * (dvdz + dwdy);
  double qx = -lam * dTdx, qy = -lam * dTdy, qz = -lam * dTdz;
  out[0] = 0.0;
  out[1] = -(txx * nx + txy * ny + txz * nz);
  out[2] = -(txy * nx + tyy * ny + tyz * nz);
  out[3] = -(txz * nx + tyz * ny + tzz * nz);
  out[4] = (-(txx * u + txy * v + txz * w) + qx) * nx + (-(txy * u + tyy * v + tyz * w) + qy) * ny +
           (-(txz * u + tyz * v + tzz * w) + qz) * nz;
}

/* _vol_index / _orient, src/operator.py:33-52 */
static inline void vol_index(int loc, int a, int b, int n, int* i, int* j, int* k) {
  int d = loc / 2;
  if (d == 0) { *i = n; *j = a; *k = b; }
  else if (d == 1) { *i = b; *j = n; *k = a; }
  else { *i = a; *j = b; *k = n; }
}
static inline void orient(int code, int a, int b, int N, int* p, int* q) {
  if (code == 1) { *p = N - a; *q = b; }
  else if (code == 2) { *p = a; *q = N - b; }
  else if (code == 3) { *p = N - a; *q = N - b; }
  else { *p = a; *q = b; }
}

#define VIDX(e, k, j, i) ((((i64)(e) * n1 + (k)) * n1 + (j)) * n1 + (i))
#define FIDX(s, q, p) ((((i64)(s)) * n1 + (q)) * n1 + (p))
#define JA(e, a, k, j, i, c) (Ja[((((((i64)(e)) * 3 + (a)) * n1 + (k)) * n1 + (j)) * n1 + (i)) * 3 + (c)])

/* k_cons_to_prim, src/operator.py:76-86 */
void orc_cons_to_prim(const double* U, double* prim, i64 n, double gamma, double R, double* mins) {
  double mr = 1e300, mp = 1e300;
#pragma omp parallel for reduction(min : mr, mp)
  for (i64 i = 0; i < n; ++i) {
    prim_point(U + i * NVAR, prim + i * NPRIM, gamma, R);
    if (prim[i * NPRIM] < mr) mr = prim[i * NPRIM];
    if (prim[i * NPRIM + 4] < mp) mp = prim[i * NPRIM + 4];
  }
  mins[0] = mr;
  mins[1] = mp;
}

/* k_viscous_contravariant, src/operator.py:89-102 (Ja in reference element layout) */
void orc_viscous_contravariant(const double* prim, const double* g, const double* Ja, double* Fvis,
                               i64 ne, int N, double gamma, double R, double Pr, double mu_ref,
                               double T_ref, int law) {
  int n1 = N + 1;
  i64 n3 = (i64)n1 * n1 * n1;
#pragma omp parallel for
  for (i64 t = 0; t < ne * n3; ++t) {
    i64 e = t / n3, node = t % n3;
    int k = (int)(node / (n1 * n1)), j = (int)((node / n1) % n1), i = (int)(node % n1);
    double mu = pt_viscosity(prim[t * NPRIM + 5], mu_ref, T_ref, law);
    double lam = pt_conductivity(mu, gamma, R, Pr);
    for (int a = 0; a < 3; ++a)
      pt_viscous_flux_dir(prim[t * NPRIM + 1], prim[t * NPRIM + 2], prim[t * NPRIM + 3], mu, lam,
                          g + t * 12, JA(e, a, k, j, i, 0), JA(e, a, k, j, i, 1), JA(e, a, k, j, i, 2),
                          Fvis + (t * 3 + a) * NVAR);
  }
}

/* k_vol_int_standard, src/operator.py:109-139 */
void orc_vol_int_standard(const double* U, const double* prim, const double* Ja, const double* Fvis,
                          const double* Dhat, double* Ut, int viscous, i64 ne, int N) {
  int n1 = N + 1;
  i64 n3 = (i64)n1 * n1 * n1;
#pragma omp parallel
  {
    double* F = (double*)malloc(sizeof(double) * n3 * 3 * NVAR);
    double f[5];
#pragma omp for
    for (i64 e = 0; e < ne; ++e) {
      for (int k = 0; k < n1; ++k)
        for (int j = 0; j < n1; ++j)
          for (int i = 0; i < n1; ++i)
            for (int a = 0; a < 3; ++a) {
              i64 t = VIDX(e, k, j, i);
              const double* pr = prim + t * NPRIM;
              pt_euler_flux_dir(pr[0], pr[1], pr[2], pr[3], pr[4], U[t * NVAR + 4], JA(e, a, k, j, i, 0),
                                JA(e, a, k, j, i, 1), JA(e, a, k, j, i, 2), f);
              for (int v = 0; v < NVAR; ++v) {
                double* dst = F + ((((i64)k * n1 + j) * n1 + i) * 3 + a) * NVAR + v;
                *dst = f[v];
                if (viscous) *dst += Fvis[(t * 3 + a) * NVAR + v];
              }
            }
#define FF(k, j, i, a, v) F[((((i64)(k) * n1 + (j)) * n1 + (i)) * 3 + (a)) * NVAR + (v)]
      for (int k = 0; k < n1; ++k)
        for (int j = 0; j < n1; ++j)
          for (int i = 0; i < n1; ++i)
            for (int v = 0; v < NVAR; ++v) {
              double acc = 0.0;
              for (int al = 0; al < n1; ++al)
                acc += Dhat[i * n1 + al] * FF(k, j, al, 0, v) + Dhat[j * n1 + al] * FF(k, al, i, 1, v) +
                       Dhat[k * n1 + al] * FF(al, j, i, 2, v);
              Ut[VIDX(e, k, j, i) * NVAR + v] += acc;
            }
#undef FF
    }
    free(F);
  }
}

/* k_vol_int_split, src/operator.py:142-209 */
void orc_vol_int_split(const double* prim, const double* Ja, const double* Fvis, const double* Dsplit,
                       double* Ut, int viscous, i64 ne, int N) {
  int n1 = N + 1;
#pragma omp parallel
  {
    double fs[5], line[16][6], met[16][3], fv[16][5], acc[16][5];
#pragma omp for
    for (i64 e = 0; e < ne; ++e) {
      for (int d = 0; d < 3; ++d)
        for (int c2 = 0; c2 < n1; ++c2)
          for (int c1 = 0; c1 < n1; ++c1) {
            int k, j, i;
            for (int m = 0; m < n1; ++m) {
              if (d == 0) { k = c2; j = c1; i = m; }
              else if (d == 1) { k = c2; j = m; i = c1; }
              else { k = m; j = c1; i = c2; }
              const double* pr = prim + VIDX(e, k, j, i) * NPRIM;
              line[m][0] = pr[0]; line[m][1] = pr[1]; line[m][2] = pr[2];
              line[m][3] = pr[3]; line[m][4] = pr[4]; line[m][5] = pr[6];
              met[m][0] = JA(e, d, k, j, i, 0);
              met[m][1] = JA(e, d, k, j, i, 1);
              met[m][2] = JA(e, d, k, j, i, 2);
              if (viscous)
                for (int v = 0; v < NVAR; ++v) fv[m][v] = Fvis[(VIDX(e, k, j, i) * 3 + d) * NVAR + v];
              for (int v = 0; v < NVAR; ++v) acc[m][v] = 0.0;
            }
            for (int m = 0; m < n1; ++m)
              for (int al = m; al < n1; ++al) {
                pt_split_flux_kep(line[m][0], line[m][1], line[m][2], line[m][3], line[m][4], line[m][5],
                                  line[al][0], line[al][1], line[al][2], line[al][3], line[al][4],
                                  line[al][5], 0.5 * (met[m][0] + met[al][0]),
                                  0.5 * (met[m][1] + met[al][1]), 0.5 * (met[m][2] + met[al][2]), fs);
                if (viscous)
                  for (int v = 0; v < NVAR; ++v) fs[v] += 0.5 * (fv[m][v] + fv[al][v]);
                if (al == m) {
                  for (int v = 0; v < NVAR; ++v) acc[m][v] += Dsplit[m * n1 + m] * fs[v];
                } else {
                  for (int v = 0; v < NVAR; ++v) {
                    acc[m][v] += Dsplit[m * n1 + al] * fs[v];
                    acc[al][v] += Dsplit[al * n1 + m] * fs[v];
                  }
                }
              }
            for (int m = 0; m < n1; ++m) {
              if (d == 0) { k = c2; j = c1; i = m; }
              else if (d == 1) { k = c2; j = m; i = c1; }
              else { k = m; j = c1; i = c2; }
              for (int v = 0; v < NVAR; ++v) Ut[VIDX(e, k, j, i) * NVAR + v] += acc[m][v];
            }
          }
    }
  }
}

/* k_prolong, src/operator.py:216-238; rows (n,5) = (side, elem, loc, is_primary, orient) */
void orc_prolong(const double* U, const i64* rows, i64 nrows, const double* l_minus, const double* l_plus,
                 int N, double* UL, double* UR) {
  int n1 = N + 1;
#pragma omp parallel for
  for (i64 r = 0; r < nrows; ++r) {
    i64 s = rows[r * 5], e = rows[r * 5 + 1];
    int loc = (int)rows[r * 5 + 2], is_p = (int)rows[r * 5 + 3], code = (int)rows[r * 5 + 4];
    const double* lv = (loc % 2 == 1) ? l_plus : l_minus;
    for (int a = 0; a < n1; ++a)
      for (int b = 0; b < n1; ++b) {
        int p, q;
        orient(code, a, b, N, &p, &q);
        for (int v = 0; v < NVAR; ++v) {
          double acc = 0.0;
          for (int m = 0; m < n1; ++m) {
            int i, j, k;
            vol_index(loc, a, b, m, &i, &j, &k);
            acc += lv[m] * U[VIDX(e, k, j, i) * NVAR + v];
          }
          (is_p == 1 ? UL : UR)[FIDX(s, q, p) * NVAR + v] = acc;
        }
      }
  }
}

/* k_prolong_grad, src/operator.py:241-266 */
void orc_prolong_grad(const double* g, const i64* rows, i64 nrows, const double* l_minus,
                      const double* l_plus, int N, double* gL, double* gR) {
  int n1 = N + 1;
#pragma omp parallel for
  for (i64 r = 0; r < nrows; ++r) {
    i64 s = rows[r * 5], e = rows[r * 5 + 1];
    int loc = (int)rows[r * 5 + 2], is_p = (int)rows[r * 5 + 3], code = (int)rows[r * 5 + 4];
    const double* lv = (loc % 2 == 1) ? l_plus : l_minus;
    double* dst = is_p == 1 ? gL : gR;
    for (int a = 0; a < n1; ++a)
      for (int b = 0; b < n1; ++b) {
        int p, q;
        orient(code, a, b, N, &p, &q);
        for (int m = 0; m < n1; ++m) {
          int i, j, k;
          vol_index(loc, a, b, m, &i, &j, &k);
          double w = lv[m];
          for (int c = 0; c < 12; ++c) {
            double* o = dst + FIDX(s, q, p) * 12 + c;
            if (m == 0) *o = w * g[VIDX(e, k, j, i) * 12 + c];
            else *o += w * g[VIDX(e, k, j, i) * 12 + c];
          }
        }
      }
  }
}

/* k_fill_flux_convective, src/operator.py:269-292; returns max bad side or -1 */
i64 orc_fill_flux_convective(const i64* sides, i64 nsides, const double* UL, const double* UR,
                             const double* nvec, const double* ssurf, double* fstar, int solver,
                             double gamma, double R, int N) {
  int n1 = N + 1;
  i64 bad = -1;
#pragma omp parallel for reduction(max : bad)
  for (i64 r = 0; r < nsides; ++r) {
    double pl[7], pr[7], f[5];
    i64 s = sides[r];
    for (int q = 0; q < n1; ++q)
      for (int p = 0; p < n1; ++p) {
        i64 fo = FIDX(s, q, p);
        prim_point(UL + fo * NVAR, pl, gamma, R);
        prim_point(UR + fo * NVAR, pr, gamma, R);
        if (pl[0] <= 0.0 || pl[4] <= 0.0 || pr[0] <= 0.0 || pr[4] <= 0.0)
          if (s > bad) bad = s;
        pt_riemann(solver, pl, UL[fo * NVAR + 4], pr, UR[fo * NVAR + 4], nvec[fo * 3], nvec[fo * 3 + 1],
                   nvec[fo * 3 + 2], gamma, f);
        for (int v = 0; v < NVAR; ++v) fstar[fo * NVAR + v] = f[v] * ssurf[fo];
      }
  }
  return bad;
}

/* k_fill_flux_viscous, src/operator.py:295-330 */
void orc_fill_flux_viscous(const i64* sides, i64 nsides, const double* UL, const double* UR,
                           const double* gL, const double* gR, const double* nvec, const double* ssurf,
                           double* fstar, double gamma, double R, double Pr, double mu_ref, double T_ref,
                           int law, int N) {
  int n1 = N + 1;
#pragma omp parallel for
  for (i64 r = 0; r < nsides; ++r) {
    double pl[7], pr[7], fl[5], fr[5];
    i64 s = sides[r];
    for (int q = 0; q < n1; ++q)
      for (int p = 0; p < n1; ++p) {
        i64 fo = FIDX(s, q, p);
        prim_point(UL + fo * NVAR, pl, gamma, R);
        prim_point(UR + fo * NVAR, pr, gamma, R);
        double nx = nvec[fo * 3], ny = nvec[fo * 3 + 1], nz = nvec[fo * 3 + 2];
        double mu = pt_viscosity(pl[5], mu_ref, T_ref, law);
        double lam = pt_conductivity(mu, gamma, R, Pr);
        pt_viscous_flux_dir(pl[1], pl[2], pl[3], mu, lam, gL + fo * 12, nx, ny, nz, fl);
        mu = pt_viscosity(pr[5], mu_ref, T_ref, law);
        lam = pt_conductivity(mu, gamma, R, Pr);
        pt_viscous_flux_dir(pr[1], pr[2], pr[3], mu, lam, gR + fo * 12, nx, ny, nz, fr);
        for (int v = 0; v < NVAR; ++v) fstar[fo * NVAR + v] += 0.5 * (fl[v] + fr[v]) * ssurf[fo];
      }
  }
}

/* k_surf_int, src/operator.py:333-358 */
void orc_surf_int(const double* fstar, const i64* ef_side, const double* ef_sign, const i64* ef_orient,
                  const double* lhat_minus, const double* lhat_plus, double* Ut, i64 ne, int N) {
  int n1 = N + 1;
#pragma omp parallel for
  for (i64 e = 0; e < ne; ++e)
    for (int k = 0; k < n1; ++k)
      for (int j = 0; j < n1; ++j)
        for (int i = 0; i < n1; ++i)
          for (int loc = 0; loc < 6; ++loc) {
            i64 s = ef_side[e * 6 + loc];
            double sign = ef_sign[e * 6 + loc];
            int code = (int)ef_orient[e * 6 + loc];
            int d = loc / 2, m, a, b, p, q;
            if (d == 0) { m = i; a = j; b = k; }
            else if (d == 1) { m = j; a = k; b = i; }
            else { m = k; a = i; b = j; }
            orient(code, a, b, N, &p, &q);
            double lh = (loc % 2 == 1) ? lhat_plus[m] : lhat_minus[m];
            double w = sign * lh;
            for (int v = 0; v < NVAR; ++v) Ut[VIDX(e, k, j, i) * NVAR + v] += w * fstar[FIDX(s, q, p) * NVAR + v];
          }
}

/* k_apply_jac, src/operator.py:361-370 */
void orc_apply_jac(double* Ut, const double* J, i64 ndof) {
#pragma omp parallel for
  for (i64 t = 0; t < ndof; ++t) {
    double w = -1.0 / J[t];
    for (int v = 0; v < NVAR; ++v) Ut[t * NVAR + v] *= w;
  }
}

/* k_lift_fill, src/operator.py:377-391 */
void orc_lift_fill(const i64* sides, i64 nsides, const double* UL, const double* UR, double* vstar,
                   double gamma, double R, int N) {
  int n1 = N + 1;
#pragma omp parallel for
  for (i64 r = 0; r < nsides; ++r) {
    double pl[7], pr[7];
    i64 s = sides[r];
    for (int q = 0; q < n1; ++q)
      for (int p = 0; p < n1; ++p) {
        i64 fo = FIDX(s, q, p);
        prim_point(UL + fo * NVAR, pl, gamma, R);
        prim_point(UR + fo * NVAR, pr, gamma, R);
        for (int l = 0; l < NLIFT; ++l) {
          int lp = l < 3 ? 1 + l : 5;
          vstar[fo * NLIFT + l] = 0.5 * (pl[lp] + pr[lp]);
        }
      }
  }
}

/* k_lift_volume, src/operator.py:394-418 */
void orc_lift_volume(const double* prim, const double* Ja, const double* Dhat, double* g, i64 ne, int N) {
  int n1 = N + 1;
#pragma omp parallel for
  for (i64 e = 0; e < ne; ++e)
    for (int k = 0; k < n1; ++k)
      for (int j = 0; j < n1; ++j)
        for (int i = 0; i < n1; ++i) {
          double* gg = g + VIDX(e, k, j, i) * 12;
          for (int c = 0; c < 12; ++c) gg[c] = 0.0;
          for (int al = 0; al < n1; ++al) {
            double di = Dhat[i * n1 + al], dj = Dhat[j * n1 + al], dk = Dhat[k * n1 + al];
            for (int d = 0; d < 3; ++d) {
              double jai = di * JA(e, 0, k, j, al, d);
              double jaj = dj * JA(e, 1, k, al, i, d);
              double jak = dk * JA(e, 2, al, j, i, d);
              for (int l = 0; l < NLIFT; ++l) {
                int lp = l < 3 ? 1 + l : 5;
                gg[d * 4 + l] += jai * prim[VIDX(e, k, j, al) * NPRIM + lp] +
                                 jaj * prim[VIDX(e, k, al, i) * NPRIM + lp] +
                                 jak * prim[VIDX(e, al, j, i) * NPRIM + lp];
              }
            }
          }
        }
}

/* k_lift_surf_and_jac, src/operator.py:421-453 */
void orc_lift_surf_and_jac(const double* vstar, const double* nvec, const double* ssurf, const i64* ef_side,
                           const double* ef_sign, const i64* ef_orient, const double* lhat_minus,
                           const double* lhat_plus, const double* J, double* g, i64 ne, int N) {
  int n1 = N + 1;
#pragma omp parallel for
  for (i64 e = 0; e < ne; ++e)
    for (int k = 0; k < n1; ++k)
      for (int j = 0; j < n1; ++j)
        for (int i = 0; i < n1; ++i) {
          double* gg = g + VIDX(e, k, j, i) * 12;
          for (int loc = 0; loc < 6; ++loc) {
            i64 s = ef_side[e * 6 + loc];
            double sign = ef_sign[e * 6 + loc];
            int code = (int)ef_orient[e * 6 + loc];
            int d = loc / 2, m, a, b, p, q;
            if (d == 0) { m = i; a = j; b = k; }
            else if (d == 1) { m = j; a = k; b = i; }
            else { m = k; a = i; b = j; }
            orient(code, a, b, N, &p, &q);
            double lh = (loc % 2 == 1) ? lhat_plus[m] : lhat_minus[m];
            i64 fo = FIDX(s, q, p);
            double w = sign * lh * ssurf[fo];
            for (int dd = 0; dd < 3; ++dd) {
              double nd = w * nvec[fo * 3 + dd];
              for (int l = 0; l < NLIFT; ++l) gg[dd * 4 + l] += nd * vstar[fo * NLIFT + l];
            }
          }
          double iw = 1.0 / J[VIDX(e, k, j, i)];
          for (int c = 0; c < 12; ++c) gg[c] *= iw;
        }
}

/* k_local_dt, src/operator.py:460-487 (serial: exact min) */
double orc_local_dt(const double* prim, const double* Ja, const double* J, i64 ne, int N, double cfl,
                    double cfl_visc, double gamma, double R, double Pr, double mu_ref, double T_ref, int law,
                    int viscous) {
  (void)R;
  int n1 = N + 1;
  i64 n3 = (i64)n1 * n1 * n1;
  double dt = 1e300;
  double scale = 2.0 * N + 1.0;
  for (i64 t = 0; t < ne * n3; ++t) {
    i64 e = t / n3, node = t % n3;
    int k = (int)(node / (n1 * n1)), j = (int)((node / n1) % n1), i = (int)(node % n1);
    const double* pr = prim + t * NPRIM;
    double a = sqrt(gamma * pr[4] / pr[0]);
    double lam = 0.0, metric2 = 0.0;
    for (int d = 0; d < 3; ++d) {
      double jx = JA(e, d, k, j, i, 0), jy = JA(e, d, k, j, i, 1), jz = JA(e, d, k, j, i, 2);
      double nrm = sqrt(jx * jx + jy * jy + jz * jz);
      double vn = pr[1] * jx + pr[2] * jy + pr[3] * jz;
      lam += fabs(vn) + a * nrm;
      metric2 += nrm * nrm;
    }
    double dta = cfl * 2.0 * J[t] / (scale * lam);
    if (dta < dt) dt = dta;
    if (viscous) {
      double mu = pt_viscosity(pr[5], mu_ref, T_ref, law);
      double nu = mu / pr[0] * pmax(4.0 / 3.0, gamma / Pr);
      if (nu > 0.0) {
        double tj = 2.0 * J[t];
        double dtv = cfl_visc * (tj * tj) / (scale * scale * metric2 * nu);
        if (dtv < dt) dt = dtv;
      }
    }
  }
  return dt;
}

/* k_indicator, src/shock.py:46-110 */
void orc_indicator(const double* U, const double* Vinv, double* alpha, double threshold, double sharpness,
                   double alpha_max, double alpha_min, double gamma, i64 ne, int N) {
  int n1 = N + 1;
  i64 n3 = (i64)n1 * n1 * n1;
#pragma omp parallel
  {
    double* ind = (double*)malloc(sizeof(double) * n3);
    double* t1 = (double*)malloc(sizeof(double) * n3);
    double* t2 = (double*)malloc(sizeof(double) * n3);
#define L3(k, j, i) ((((i64)(k)) * n1 + (j)) * n1 + (i))
#pragma omp for
    for (i64 e = 0; e < ne; ++e) {
      for (int k = 0; k < n1; ++k)
        for (int j = 0; j < n1; ++j)
          for (int i = 0; i < n1; ++i) {
            const double* u = U + VIDX(e, k, j, i) * NVAR;
            double rho = u[0];
            double p = (gamma - 1.0) * (u[4] - 0.5 * (u[1] * u[1] + u[2] * u[2] + u[3] * u[3]) / rho);
            ind[L3(k, j, i)] = rho * p;
          }
      for (int k = 0; k < n1; ++k)
        for (int j = 0; j < n1; ++j)
          for (int i = 0; i < n1; ++i) {
            double acc = 0.0;
            for (int m = 0; m < n1; ++m) acc += Vinv[i * n1 + m] * ind[L3(k, j, m)];
            t1[L3(k, j, i)] = acc;
          }
      for (int k = 0; k < n1; ++k)
        for (int i = 0; i < n1; ++i)
          for (int j = 0; j < n1; ++j) {
            double acc = 0.0;
            for (int m = 0; m < n1; ++m) acc += Vinv[j * n1 + m] * t1[L3(k, m, i)];
            t2[L3(k, j, i)] = acc;
          }
      for (int j = 0; j < n1; ++j)
        for (int i = 0; i < n1; ++i)
          for (int k = 0; k < n1; ++k) {
            double acc = 0.0;
            for (int m = 0; m < n1; ++m) acc += Vinv[k * n1 + m] * t2[L3(m, j, i)];
            t1[L3(k, j, i)] = acc;
          }
      double total = 0.0, clip1 = 0.0, clip2 = 0.0;
      for (int k = 0; k < n1; ++k)
        for (int j = 0; j < n1; ++j)
          for (int i = 0; i < n1; ++i) {
            double m2 = t1[L3(k, j, i)] * t1[L3(k, j, i)];
            total += m2;
            if (k < N && j < N && i < N) clip1 += m2;
            if (k < N - 1 && j < N - 1 && i < N - 1) clip2 += m2;
          }
      double energy = 0.0;
      if (total > 1e-300) energy = (total - clip1) / total;
      if (clip1 > 1e-300) {
        double e2 = (clip1 - clip2) / clip1;
        if (e2 > energy) energy = e2;
      }
      double a = 1.0 / (1.0 + exp(-sharpness / threshold * (energy - threshold)));
      if (a > alpha_max) a = alpha_max;
      if (a < alpha_min) a = 0.0;
      alpha[e] = a;
    }
#undef L3
    free(ind);
    free(t1);
    free(t2);
  }
}

/* k_fv_residual, src/shock.py:113-195 (flagged elements are disjoint: parallel over them) */
void orc_fv_residual(const i64* flagged, i64 nf, const double* U, const double* fvm0, const double* fvm1,
                     const double* fvm2, const double* weights, const double* J, const double* fstar,
                     const i64* ef_side, const double* ef_sign, const i64* ef_orient, int solver,
                     double gamma, double R, double* RFV, int N) {
  int n1 = N + 1;
#define FVM(arr, e, r1, r2, h, c) (arr[(((((i64)(e)) * n1 + (r1)) * n1 + (r2)) * (n1 + 1) + (h)) * 3 + (c)])
#pragma omp parallel
  {
    double pl[7], pr[7], f[5];
    double Fline[17][5];
#pragma omp for
    for (i64 idx = 0; idx < nf; ++idx) {
      i64 e = flagged[idx];
      for (int v = 0; v < NVAR; ++v)
        for (int k = 0; k < n1; ++k)
          for (int j = 0; j < n1; ++j)
            for (int i = 0; i < n1; ++i) RFV[VIDX(e, k, j, i) * NVAR + v] = 0.0;
      for (int d = 0; d < 3; ++d) {
        int loc_m = 2 * d, loc_p = 2 * d + 1;
        i64 s_m = ef_side[e * 6 + loc_m], s_p = ef_side[e * 6 + loc_p];
        double sg_m = ef_sign[e * 6 + loc_m], sg_p = ef_sign[e * 6 + loc_p];
        int cd_m = (int)ef_orient[e * 6 + loc_m], cd_p = (int)ef_orient[e * 6 + loc_p];
        for (int a = 0; a < n1; ++a)
          for (int b = 0; b < n1; ++b) {
            int p, q;
            orient(cd_m, a, b, N, &p, &q);
            for (int v = 0; v < NVAR; ++v) Fline[0][v] = -sg_m * fstar[FIDX(s_m, q, p) * NVAR + v];
            orient(cd_p, a, b, N, &p, &q);
            for (int v = 0; v < NVAR; ++v) Fline[n1][v] = sg_p * fstar[FIDX(s_p, q, p) * NVAR + v];
            for (int h = 1; h < n1; ++h) {
              int iL[3], iR[3];
              double mx, my, mz;
              if (d == 0) {
                iL[0] = h - 1; iL[1] = a; iL[2] = b; iR[0] = h; iR[1] = a; iR[2] = b;
                mx = FVM(fvm0, e, b, a, h, 0); my = FVM(fvm0, e, b, a, h, 1); mz = FVM(fvm0, e, b, a, h, 2);
              } else if (d == 1) {
                iL[0] = b; iL[1] = h - 1; iL[2] = a; iR[0] = b; iR[1] = h; iR[2] = a;
                mx = FVM(fvm1, e, a, b, h, 0); my = FVM(fvm1, e, a, b, h, 1); mz = FVM(fvm1, e, a, b, h, 2);
              } else {
                iL[0] = a; iL[1] = b; iL[2] = h - 1; iR[0] = a; iR[1] = b; iR[2] = h;
                mx = FVM(fvm2, e, b, a, h, 0); my = FVM(fvm2, e, b, a, h, 1); mz = FVM(fvm2, e, b, a, h, 2);
              }
              double snorm = sqrt(mx * mx + my * my + mz * mz);
              double nx = mx / snorm, ny = my / snorm, nz = mz / snorm;
              const double* uL = U + VIDX(e, iL[2], iL[1], iL[0]) * NVAR;
              const double* uR = U + VIDX(e, iR[2], iR[1], iR[0]) * NVAR;
              prim_point(uL, pl, gamma, R);
              prim_point(uR, pr, gamma, R);
              pt_riemann(solver, pl, uL[4], pr, uR[4], nx, ny, nz, gamma, f);
              for (int v = 0; v < NVAR; ++v) Fline[h][v] = f[v] * snorm;
            }
            for (int h = 0; h < n1; ++h) {
              double iw = 1.0 / weights[h];
              int i, j, k;
              if (d == 0) { i = h; j = a; k = b; }
              else if (d == 1) { i = b; j = h; k = a; }
              else { i = a; j = b; k = h; }
              for (int v = 0; v < NVAR; ++v)
                RFV[VIDX(e, k, j, i) * NVAR + v] -= (Fline[h + 1][v] - Fline[h][v]) * iw;
            }
          }
      }
      for (int k = 0; k < n1; ++k)
        for (int j = 0; j < n1; ++j)
          for (int i = 0; i < n1; ++i) {
            double iw = 1.0 / J[VIDX(e, k, j, i)];
            for (int v = 0; v < NVAR; ++v) RFV[VIDX(e, k, j, i) * NVAR + v] *= iw;
          }
    }
  }
#undef FVM
}

/* k_blend, src/shock.py:198-210 */
void orc_blend(const i64* flagged, i64 nf, const double* alpha, double* Ut, const double* RFV, int N) {
  int n1 = N + 1;
  i64 n3 = (i64)n1 * n1 * n1;
#pragma omp parallel for
  for (i64 idx = 0; idx < nf; ++idx) {
    i64 e = flagged[idx];
    double a = alpha[e];
    double b = 1.0 - a;
    for (i64 t = e * n3 * NVAR; t < (e + 1) * n3 * NVAR; ++t) Ut[t] = b * Ut[t] + a * RFV[t];
  }
}

/* k_mms_source, src/testcases.py:51-70 */
void orc_mms_source(const double* x, double t, double* Ut, i64 n, double A, double a, double gamma,
                    double mu, double Pr) {
  const double W = 2.0 * 3.141592653589793;
  double c_mom = 0.5 * (5.0 * gamma + 1.0) - a;
  double c_e1 = A * (3.0 * gamma - a);
  double c_e2 = 7.5 * gamma + 4.5 - 4.0 * a;
  double c_e3 = 3.0 * W * gamma * mu / Pr;
  for (i64 i = 0; i < n; ++i) {
    double ph = W * (x[i * 3] + x[i * 3 + 1] + x[i * 3 + 2] - a * t);
    double sn = sin(ph), cs = cos(ph);
    double aw = A * W;
    double s_mom = aw * cs * (2.0 * A * (gamma - 1.0) * sn + c_mom);
    Ut[i * 5 + 0] += aw * (3.0 - a) * cs;
    Ut[i * 5 + 1] += s_mom;
    Ut[i * 5 + 2] += s_mom;
    Ut[i * 5 + 3] += s_mom;
    Ut[i * 5 + 4] += aw * (c_e1 * 2.0 * sn * cs + c_e2 * cs + c_e3 * sn);
  }
}

/* rk_step numpy update, src/timedisc.py:132-137 */
void orc_lserk(double* U, double* work, const double* Ut, i64 n, double A, double B, double dt, int first) {
#pragma omp parallel for
  for (i64 t = 0; t < n; ++t) {
    if (first) work[t] = dt * Ut[t];
    else {
      work[t] *= A;
      work[t] += dt * Ut[t];
    }
    U[t] += B * work[t];
  }
}

/* k_analysis_partials, src/testcases.py:190-226 (per element, nodes in (k,j,i)
 * order; g may be NULL when !viscous) */
void orc_analysis_partials(const double* U, const double* g, const double* J, const double* w,
                           double gamma, double R, double mu_ref, double T_ref, int law, double mu0,
                           int viscous, double* out, i64 ne, int N) {
  int n1 = N + 1;
#pragma omp parallel for
  for (i64 e = 0; e < ne; ++e) {
    double* o = out + e * 9;
    for (int v = 0; v < 9; ++v) o[v] = 0.0;
    for (int k = 0; k < n1; ++k)
      for (int j = 0; j < n1; ++j)
        for (int i = 0; i < n1; ++i) {
          i64 t = VIDX(e, k, j, i);
          double dv = J[t] * w[i] * w[j] * w[k];
          const double* u = U + t * NVAR;
          double rho = u[0], mx = u[1], my = u[2], mz = u[3];
          o[0] += dv * rho;
          o[1] += dv * mx;
          o[2] += dv * my;
          o[3] += dv * mz;
          o[4] += dv * u[4];
          o[5] += dv * (mx * mx + my * my + mz * mz) / rho;
          if (viscous) {
            double p = (gamma - 1.0) * (u[4] - 0.5 * (mx * mx + my * my + mz * mz) / rho);
            double T = p / (rho * R);
            double mu = pt_viscosity(T, mu_ref, T_ref, law) / mu0;
            const double* gg = g + t * 12;
            double wx = gg[6] - gg[9], wy = gg[8] - gg[2], wz = gg[1] - gg[4];
            double dvg = gg[0] + gg[5] + gg[10];
            o[6] += dv * mu * (wx * wx + wy * wy + wz * wz);
            o[7] += dv * mu * dvg * dvg;
          }
          o[8] += dv;
        }
  }
}
