// Pointwise gas dynamics for the DGSEM hot path (device, inlined).
//
// Every routine evaluates the same IEEE float64 operations in the same order
// as the reference point routine it cites (reference src/equations.py and
// src/operator.py). Compiled with -fmad=false (the "exact" kernel set) the
// results are bit-identical to the reference's numba kernels; the "fast" set
// is the same source with FMA contraction enabled.
#pragma once
#include <cstdint>

namespace hdg {

struct Gas {
  double gamma, R, Pr, mu_ref, T_ref;
  int law;  // 0 constant viscosity, 1 Sutherland
};

__device__ __forceinline__ double dmax(double a, double b) { return (b > a) ? b : a; }  // python max(a, b)
__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }  // python min(a, b)

// _prim_point (src/operator.py:55-69): (rho, u, v, w, p, T, h)
__device__ __forceinline__ void prim_point(const double U[5], double o[7], const Gas& g) {
  const double rho = U[0];
  const double ir = 1.0 / rho;
  const double u = U[1] * ir, v = U[2] * ir, w = U[3] * ir;
  const double p = (g.gamma - 1.0) * (U[4] - 0.5 * rho * (u * u + v * v + w * w));
  o[0] = rho; o[1] = u; o[2] = v; o[3] = w; o[4] = p;
  o[5] = p * ir / g.R;
  o[6] = (U[4] + p) * ir;
}

// pt_viscosity / pt_conductivity (src/equations.py:75-85)
__device__ __forceinline__ double viscosity(double T, const Gas& g) {
  if (g.law == 0) return g.mu_ref;
  const double tr = T / g.T_ref;
  return g.mu_ref * 1.4042 * tr * sqrt(tr) / (tr + 0.4042);
}
__device__ __forceinline__ double conductivity(double mu, const Gas& g) {
  return g.gamma * g.R / (g.gamma - 1.0) * mu / g.Pr;
}
__device__ __forceinline__ double sound_speed(double rho, double p, double gamma) {
  return sqrt(gamma * p / rho);
}

// pt_euler_flux_dir (src/equations.py:93-102)
__device__ __forceinline__ void euler_flux_dir(double rho, double u, double v, double w, double p,
                                               double rhoE, double nx, double ny, double nz,
                                               double out[5]) {
  const double vn = u * nx + v * ny + w * nz;
  const double m = rho * vn;
  out[0] = m;
  out[1] = m * u + p * nx;
  out[2] = m * v + p * ny;
  out[3] = m * w + p * nz;
  out[4] = vn * (rhoE + p);
}

// pt_split_flux_kep (src/equations.py:235-259): symmetric in (L, R) bit for bit
__device__ __forceinline__ void kep_flux(double rL, double uL, double vL, double wL, double pL, double hL,
                                         double rR, double uR, double vR, double wR, double pR, double hR,
                                         double jx, double jy, double jz, double out[5]) {
  const double rm = 0.5 * (rL + rR);
  const double um = 0.5 * (uL + uR);
  const double vm = 0.5 * (vL + vR);
  const double wm = 0.5 * (wL + wR);
  const double pm = 0.5 * (pL + pR);
  const double hm = 0.5 * (hL + hR);
  const double vn = um * jx + vm * jy + wm * jz;
  const double m = rm * vn;
  out[0] = m;
  out[1] = m * um + pm * jx;
  out[2] = m * vm + pm * jy;
  out[3] = m * wm + pm * jz;
  out[4] = m * hm;
}

// kep_flux on pre-halved node states and metrics: the arithmetic means become
// plain sums, 0.5*(a+b) == 0.5*a + 0.5*b exactly (binary scaling), so the result
// is bitwise the reference's (element kernel split-form pair loop)
__device__ __forceinline__ void kep_flux_half(double rL, double uL, double vL, double wL,
                                              double pL, double hL, double rR, double uR,
                                              double vR, double wR, double pR, double hR,
                                              double jx, double jy, double jz, double out[5]) {
  const double rm = rL + rR;
  const double um = uL + uR;
  const double vm = vL + vR;
  const double wm = wL + wR;
  const double pm = pL + pR;
  const double hm = hL + hR;
  const double vn = um * jx + vm * jy + wm * jz;
  const double m = rm * vn;
  out[0] = m;
  out[1] = m * um + pm * jx;
  out[2] = m * vm + pm * jy;
  out[3] = m * wm + pm * jz;
  out[4] = m * hm;
}

// pt_llf (src/equations.py:105-121)
__device__ __forceinline__ void llf(const double* L, double rhoEL, const double* R, double rhoER,
                                    double nx, double ny, double nz, double gamma, double out[5]) {
  double fR[5];
  euler_flux_dir(L[0], L[1], L[2], L[3], L[4], rhoEL, nx, ny, nz, out);
  euler_flux_dir(R[0], R[1], R[2], R[3], R[4], rhoER, nx, ny, nz, fR);
  const double vnL = L[1] * nx + L[2] * ny + L[3] * nz;
  const double vnR = R[1] * nx + R[2] * ny + R[3] * nz;
  const double lam = dmax(fabs(vnL) + sound_speed(L[0], L[4], gamma),
                          fabs(vnR) + sound_speed(R[0], R[4], gamma));
  out[0] = 0.5 * (out[0] + fR[0]) - 0.5 * lam * (R[0] - L[0]);
  out[1] = 0.5 * (out[1] + fR[1]) - 0.5 * lam * (R[0] * R[1] - L[0] * L[1]);
  out[2] = 0.5 * (out[2] + fR[2]) - 0.5 * lam * (R[0] * R[2] - L[0] * L[2]);
  out[3] = 0.5 * (out[3] + fR[3]) - 0.5 * lam * (R[0] * R[3] - L[0] * L[3]);
  out[4] = 0.5 * (out[4] + fR[4]) - 0.5 * lam * (rhoER - rhoEL);
}

// pt_hllc (src/equations.py:124-185)
__device__ __forceinline__ void hllc(const double* L, double rhoEL, const double* R, double rhoER,
                                     double nx, double ny, double nz, double gamma, double out[5]) {
  const double rhoL = L[0], uL = L[1], vL = L[2], wL = L[3], pL = L[4];
  const double rhoR = R[0], uR = R[1], vR = R[2], wR = R[3], pR = R[4];
  const double vnL = uL * nx + vL * ny + wL * nz;
  const double vnR = uR * nx + vR * ny + wR * nz;
  const double aL = sound_speed(rhoL, pL, gamma);
  const double aR = sound_speed(rhoR, pR, gamma);
  const double sqL = sqrt(rhoL), sqR = sqrt(rhoR);
  const double fac = 1.0 / (sqL + sqR);
  const double vnRoe = (sqL * vnL + sqR * vnR) * fac;
  const double HL = (rhoEL + pL) / rhoL;
  const double HR = (rhoER + pR) / rhoR;
  const double HRoe = (sqL * HL + sqR * HR) * fac;
  const double u2Roe = ((sqL * (uL * uL + vL * vL + wL * wL) + sqR * (uR * uR + vR * vR + wR * wR)) * fac);
  const double aRoe = sqrt(dmax((gamma - 1.0) * (HRoe - 0.5 * u2Roe), 1e-300));
  const double sL = dmin(vnL - aL, vnRoe - aRoe);
  const double sR = dmax(vnR + aR, vnRoe + aRoe);
  if (sL >= 0.0) { euler_flux_dir(rhoL, uL, vL, wL, pL, rhoEL, nx, ny, nz, out); return; }
  if (sR <= 0.0) { euler_flux_dir(rhoR, uR, vR, wR, pR, rhoER, nx, ny, nz, out); return; }
  const double sM = (pR - pL + rhoL * vnL * (sL - vnL) - rhoR * vnR * (sR - vnR)) /
                    (rhoL * (sL - vnL) - rhoR * (sR - vnR));
  if (sM >= 0.0) {
    euler_flux_dir(rhoL, uL, vL, wL, pL, rhoEL, nx, ny, nz, out);
    const double rho_s = rhoL * (sL - vnL) / (sL - sM);
    const double d = sM - vnL;
    const double us0 = rho_s;
    const double us1 = rho_s * (uL + d * nx);
    const double us2 = rho_s * (vL + d * ny);
    const double us3 = rho_s * (wL + d * nz);
    const double us4 = rho_s * (rhoEL / rhoL + d * (sM + pL / (rhoL * (sL - vnL))));
    out[0] += sL * (us0 - rhoL);
    out[1] += sL * (us1 - rhoL * uL);
    out[2] += sL * (us2 - rhoL * vL);
    out[3] += sL * (us3 - rhoL * wL);
    out[4] += sL * (us4 - rhoEL);
  } else {
    euler_flux_dir(rhoR, uR, vR, wR, pR, rhoER, nx, ny, nz, out);
    const double rho_s = rhoR * (sR - vnR) / (sR - sM);
    const double d = sM - vnR;
    const double us0 = rho_s;
    const double us1 = rho_s * (uR + d * nx);
    const double us2 = rho_s * (vR + d * ny);
    const double us3 = rho_s * (wR + d * nz);
    const double us4 = rho_s * (rhoER / rhoR + d * (sM + pR / (rhoR * (sR - vnR))));
    out[0] += sR * (us0 - rhoR);
    out[1] += sR * (us1 - rhoR * uR);
    out[2] += sR * (us2 - rhoR * vR);
    out[3] += sR * (us3 - rhoR * wR);
    out[4] += sR * (us4 - rhoER);
  }
}

// pt_llf_split (src/equations.py:188-210): LLF dissipation around the KEP central flux
__device__ __forceinline__ void llf_split(const double* L, double rhoEL, const double* R, double rhoER,
                                          double nx, double ny, double nz, double gamma, double out[5]) {
  kep_flux(L[0], L[1], L[2], L[3], L[4], (rhoEL + L[4]) / L[0],
           R[0], R[1], R[2], R[3], R[4], (rhoER + R[4]) / R[0], nx, ny, nz, out);
  const double vnL = L[1] * nx + L[2] * ny + L[3] * nz;
  const double vnR = R[1] * nx + R[2] * ny + R[3] * nz;
  const double lam = dmax(fabs(vnL) + sound_speed(L[0], L[4], gamma),
                          fabs(vnR) + sound_speed(R[0], R[4], gamma));
  out[0] -= 0.5 * lam * (R[0] - L[0]);
  out[1] -= 0.5 * lam * (R[0] * R[1] - L[0] * L[1]);
  out[2] -= 0.5 * lam * (R[0] * R[2] - L[0] * L[2]);
  out[3] -= 0.5 * lam * (R[0] * R[3] - L[0] * L[3]);
  out[4] -= 0.5 * lam * (rhoER - rhoEL);
}

enum { RIEMANN_LLF = 0, RIEMANN_HLLC = 1, RIEMANN_LLF_SPLIT = 2 };

// pt_riemann (src/equations.py:219-232); L, R are 7-prim arrays (rho,u,v,w,p,...)
__device__ __forceinline__ void riemann(int solver, const double* L, double rhoEL, const double* R,
                                        double rhoER, double nx, double ny, double nz, double gamma,
                                        double out[5]) {
  if (solver == RIEMANN_HLLC) hllc(L, rhoEL, R, rhoER, nx, ny, nz, gamma, out);
  else if (solver == RIEMANN_LLF_SPLIT) llf_split(L, rhoEL, R, rhoER, nx, ny, nz, gamma, out);
  else llf(L, rhoEL, R, rhoER, nx, ny, nz, gamma, out);
}

// pt_viscous_flux_dir (src/equations.py:262-285); g[d*4 + l], d = d/dx,y,z, l = u,v,w,T.
// Writes out[1..4]; out[0] is identically zero.
__device__ __forceinline__ void viscous_flux_dir(double u, double v, double w, double mu, double lam,
                                                 const double* g, double nx, double ny, double nz,
                                                 double out[5]) {
  const double dudx = g[0], dvdx = g[1], dwdx = g[2], dTdx = g[3];
  const double dudy = g[4], dvdy = g[5], dwdy = g[6], dTdy = g[7];
  const double dudz = g[8], dvdz = g[9], dwdz = g[10], dTdz = g[11];
  const double divu = dudx + dvdy + dwdz;
  const double txx = mu * (2.0 * dudx - 2.0 / 3.0 * divu);
  const double tyy = mu * (2.0 * dvdy - 2.0 / 3.0 * divu);
  const double tzz = mu * (2.0 * dwdz - 2.0 / 3.0 * divu);
  const double txy = mu * (dudy + dvdx);
  const double txz = mu * (dudz + dwdx);
  const double tyz = mu * (dvdz + dwdy);
  const double qx = -lam * dTdx, qy = -lam * dTdy, qz = -lam * dTdz;
  out[0] = 0.0;
  out[1] = -(txx * nx + txy * ny + txz * nz);
  out[2] = -(txy * nx + tyy * ny + tyz * nz);
  out[3] = -(txz * nx + tyz * ny + tzz * nz);
  out[4] = (-(txx * u + txy * v + txz * w) + qx) * nx + (-(txy * u + tyy * v + tyz * w) + qy) * ny +
           (-(txz * u + tyz * v + tzz * w) + qz) * nz;
}

}  // namespace hdg
