"""ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).

CPU restatement of the reference's hot path: the C kernels in
``hexdg_oracle.c`` (one per reference numba kernel, same operation order,
bit-identical results) driven in the reference's single-rank task order
(``RankWorker._build_rhs``, reference src/parallel.py:399-517) and the
reference ``rk_step`` / ``_compute_dt`` (src/timedisc.py:114-138,
src/parallel.py:595-604).

Pinned: tests/test_oracle_golden.py checks every function here against golden
vectors produced by the reference package itself (tests/golden/make_golden.py).
The product path never imports this package.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "hexdg_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
LIB_EXT = os.path.join(HERE, "liboracle_ld.so")
CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
          "-std=c11"]
# extended precision (hexdg_oracle_ld.c): the same source with every double an x87
# long double (64-bit significand), <tgmath.h> routing the math functions to their
# long double forms. Not bitwise anything: an accurate yardstick for the
# floating-point error of the reference itself and of the FMA kernel set on
# ill-conditioned (low-Mach) cases.
SRC_EXT = os.path.join(HERE, "hexdg_oracle_ld.c")
FT = np.float64           # the oracle's array type (np.longdouble in extended mode)
_ext = False

RIEMANN_LLF, RIEMANN_HLLC, RIEMANN_LLF_SPLIT = 0, 1, 2


def build(force=False, extended=False):
    lib_path, src = (LIB_EXT, SRC_EXT) if extended else (LIB, SRC)
    if force or not os.path.exists(lib_path) or os.path.getmtime(lib_path) < max(
            os.path.getmtime(SRC), os.path.getmtime(src)):
        subprocess.run(["gcc"] + CFLAGS + [src, "-o", lib_path, "-lm"], check=True)
    return lib_path


def extended(on=True):
    """Switch this module to the long double build (arrays np.longdouble) or back."""
    global _lib, FT, D, _ext
    if on != _ext:
        _lib = None
    _ext = bool(on)
    FT = np.longdouble if on else np.float64
    D = ctypes.c_longdouble if on else ctypes.c_double


_lib = None
D, I = ctypes.c_double, ctypes.c_int64
P = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build(extended=_ext))
        sig = {
            "orc_cons_to_prim": [P, P, I, D, D, P],
            "orc_viscous_contravariant": [P, P, P, P, I, ctypes.c_int, D, D, D, D, D, ctypes.c_int],
            "orc_vol_int_standard": [P, P, P, P, P, P, ctypes.c_int, I, ctypes.c_int],
            "orc_vol_int_split": [P, P, P, P, P, ctypes.c_int, I, ctypes.c_int],
            "orc_prolong": [P, P, I, P, P, ctypes.c_int, P, P],
            "orc_prolong_grad": [P, P, I, P, P, ctypes.c_int, P, P],
            "orc_fill_flux_convective": [P, I, P, P, P, P, P, ctypes.c_int, D, D, ctypes.c_int],
            "orc_fill_flux_viscous": [P, I, P, P, P, P, P, P, P, D, D, D, D, D, ctypes.c_int,
                                      ctypes.c_int],
            "orc_surf_int": [P, P, P, P, P, P, P, I, ctypes.c_int],
            "orc_apply_jac": [P, P, I],
            "orc_lift_fill": [P, I, P, P, P, D, D, ctypes.c_int],
            "orc_lift_volume": [P, P, P, P, I, ctypes.c_int],
            "orc_lift_surf_and_jac": [P, P, P, P, P, P, P, P, P, P, I, ctypes.c_int],
            "orc_local_dt": [P, P, P, I, ctypes.c_int, D, D, D, D, D, D, D, ctypes.c_int,
                             ctypes.c_int],
            "orc_indicator": [P, P, P, D, D, D, D, D, I, ctypes.c_int],
            "orc_fv_residual": [P, I, P, P, P, P, P, P, P, P, P, P, ctypes.c_int, D, D, P,
                                ctypes.c_int],
            "orc_blend": [P, I, P, P, P, ctypes.c_int],
            "orc_mms_source": [P, D, P, I, D, D, D, D, D],
            "orc_lserk": [P, P, P, I, D, D, D, ctypes.c_int],
            "orc_analysis_partials": [P, P, P, P, D, D, D, D, ctypes.c_int, D, ctypes.c_int, P, I,
                                      ctypes.c_int],
        }
        for name, args in sig.items():
            getattr(L, name).argtypes = args
        L.orc_fill_flux_convective.restype = ctypes.c_int64
        L.orc_local_dt.restype = D
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f(a):
    return np.ascontiguousarray(a, dtype=FT)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def modal_threshold(N):
    return 0.5 * 10.0 ** (-1.8 * (N + 1.0) ** 0.25)   # src/shock.py:41-43


SHARPNESS = float(np.log(1.0 / 1e-4 - 1.0))            # src/shock.py:29


def subcell_interface_metrics(Ja, weights, D):
    """src/shock.py:213-257 (numpy, as the reference: host setup)."""
    n1 = D.shape[0]
    ne = Ja.shape[0]
    w = weights
    dJ0 = np.einsum("im,ekjmc->ekjic", D, Ja[:, 0])
    fvm0 = np.empty((ne, n1, n1, n1 + 1, 3), dtype=FT)
    fvm0[..., 0, :] = Ja[:, 0][:, :, :, 0, :]
    for h in range(n1):
        fvm0[..., h + 1, :] = fvm0[..., h, :] + w[h] * dJ0[..., h, :]
    dJ1 = np.einsum("jm,ekmic->ekjic", D, Ja[:, 1])
    fvm1 = np.empty((ne, n1, n1, n1 + 1, 3), dtype=FT)
    acc = Ja[:, 1][:, :, 0, :, :].copy()
    fvm1[:, :, :, 0, :] = acc
    for h in range(n1):
        acc = acc + w[h] * dJ1[:, :, h, :, :]
        fvm1[:, :, :, h + 1, :] = acc
    dJ2 = np.einsum("km,emjic->ekjic", D, Ja[:, 2])
    fvm2 = np.empty((ne, n1, n1, n1 + 1, 3), dtype=FT)
    acc = Ja[:, 2][:, 0, :, :, :].copy()
    fvm2[:, :, :, 0, :] = acc
    for h in range(n1):
        acc = acc + w[h] * dJ2[:, h, :, :, :]
        fvm2[:, :, :, h + 1, :] = acc
    return fvm0, np.ascontiguousarray(fvm1), np.ascontiguousarray(fvm2)


class OracleDomain:
    """Arrays of one single-rank domain in the reference's layouts.

    ``src`` is any object with the reference Domain attribute names (the
    product Domain's host mirrors, or a golden fixture namespace).
    """

    def __init__(self, src, basis, gas):
        self.N = basis.N
        self.n1 = basis.N + 1
        self.basis = basis
        self.gas = gas
        self.ne = int(src.ef_side.shape[0])
        self.ns = int(src.ssurf.shape[0])
        self.Ja = _f(src.Ja)
        self.J = _f(src.J)
        self.x = _f(src.x)
        self.nvec = _f(src.nvec)
        self.ssurf = _f(src.ssurf)
        self.ef_side = _i(src.ef_side)
        self.ef_sign = _f(src.ef_sign)
        self.ef_orient = _i(src.ef_orient)
        self.rows_inner = _i(src.rows_inner).reshape(-1, 5)
        self.sides_inner = _i(src.sides_inner)
        self.sides_bc = _i(src.sides_bc)
        self.side_bc = _i(src.side_bc)
        self.bc_states = _f(src.bc_states).reshape(8, 5)
        n1, ne, ns = self.n1, self.ne, self.ns
        self.U = np.zeros((ne, n1, n1, n1, 5), dtype=FT)
        self.prim = np.zeros((ne, n1, n1, n1, 7), dtype=FT)
        self.Ut = np.zeros_like(self.U)
        self.UL = np.zeros((ns, n1, n1, 5), dtype=FT)
        self.UR = np.zeros_like(self.UL)
        self.fstar = np.zeros_like(self.UL)
        self.viscous = gas.mu_ref > 0.0
        self.g = np.zeros((ne, n1, n1, n1, 3, 4), dtype=FT)
        self.gL = np.zeros((ns, n1, n1, 3, 4), dtype=FT)
        self.gR = np.zeros_like(self.gL)
        self.vstar = np.zeros((ns, n1, n1, 4), dtype=FT)
        self.Fvis = np.zeros((ne, n1, n1, n1, 3, 5), dtype=FT)
        self.alpha = np.zeros(ne, dtype=FT)
        self._fvm = None

    # individual kernels ------------------------------------------------------
    def cons_to_prim(self):
        mins = np.zeros(2, dtype=FT)
        lib().orc_cons_to_prim(_p(self.U), _p(self.prim), self.U.size // 5, self.gas.gamma,
                               self.gas.R, _p(mins))
        return mins

    def prolong(self):
        b = self.basis
        lib().orc_prolong(_p(self.U), _p(self.rows_inner), self.rows_inner.shape[0],
                          _p(_f(b.l_minus)), _p(_f(b.l_plus)), self.N, _p(self.UL), _p(self.UR))
        for sl in self.sides_bc:
            self.UR[sl] = self.bc_states[self.side_bc[sl]]

    def fill_flux(self, solver):
        g = self.gas
        s = self.sides_inner
        bad = lib().orc_fill_flux_convective(_p(s), s.size, _p(self.UL), _p(self.UR), _p(self.nvec),
                                             _p(self.ssurf), _p(self.fstar), solver, g.gamma, g.R,
                                             self.N)
        if self.viscous:
            lib().orc_fill_flux_viscous(_p(s), s.size, _p(self.UL), _p(self.UR), _p(self.gL),
                                        _p(self.gR), _p(self.nvec), _p(self.ssurf), _p(self.fstar),
                                        g.gamma, g.R, g.Pr, g.mu_ref, g.T_ref,
                                        int(g.viscosity_law), self.N)
        return bad

    def lift(self):
        g, b = self.gas, self.basis
        s = self.sides_inner
        L = lib()
        L.orc_lift_fill(_p(s), s.size, _p(self.UL), _p(self.UR), _p(self.vstar), g.gamma, g.R,
                        self.N)
        L.orc_lift_volume(_p(self.prim), _p(self.Ja), _p(_f(b.Dhat)), _p(self.g), self.ne, self.N)
        L.orc_lift_surf_and_jac(_p(self.vstar), _p(self.nvec), _p(self.ssurf), _p(self.ef_side),
                                _p(self.ef_sign), _p(self.ef_orient), _p(_f(b.lhat_minus)),
                                _p(_f(b.lhat_plus)), _p(self.J), _p(self.g), self.ne, self.N)
        L.orc_viscous_contravariant(_p(self.prim), _p(self.g), _p(self.Ja), _p(self.Fvis), self.ne,
                                    self.N, g.gamma, g.R, g.Pr, g.mu_ref, g.T_ref,
                                    int(g.viscosity_law))
        L.orc_prolong_grad(_p(self.g), _p(self.rows_inner), self.rows_inner.shape[0],
                           _p(_f(b.l_minus)), _p(_f(b.l_plus)), self.N, _p(self.gL), _p(self.gR))
        for sl in self.sides_bc:
            self.gR[sl] = self.gL[sl]

    def vol_int(self, split):
        b = self.basis
        if split:
            lib().orc_vol_int_split(_p(self.prim), _p(self.Ja), _p(self.Fvis), _p(_f(b.Dsplit)),
                                    _p(self.Ut), int(self.viscous), self.ne, self.N)
        else:
            lib().orc_vol_int_standard(_p(self.U), _p(self.prim), _p(self.Ja), _p(self.Fvis),
                                       _p(_f(b.Dhat)), _p(self.Ut), int(self.viscous), self.ne,
                                       self.N)

    def surf_int(self, fstar=None, Ut=None):
        b = self.basis
        fs = self.fstar if fstar is None else _f(fstar)
        ut = self.Ut if Ut is None else Ut
        lib().orc_surf_int(_p(fs), _p(self.ef_side), _p(self.ef_sign), _p(self.ef_orient),
                           _p(_f(b.lhat_minus)), _p(_f(b.lhat_plus)), _p(ut), self.ne, self.N)
        return ut

    def apply_jac(self):
        lib().orc_apply_jac(_p(self.Ut), _p(self.J), self.ne * self.n1 ** 3)

    def fvm(self):
        if self._fvm is None:
            b = self.basis
            self._fvm = subcell_interface_metrics(self.Ja, b.weights, b.D)
        return self._fvm

    def indicator(self, shock):
        N = self.N
        if shock["constant"]:
            self.alpha[:] = min(shock["alpha_const"], shock["alpha_max"])
        else:
            lib().orc_indicator(_p(self.U), _p(_f(self.basis.vandermonde_modal)), _p(self.alpha),
                                modal_threshold(N), SHARPNESS, shock["alpha_max"],
                                shock["alpha_min"], self.gas.gamma, self.ne, N)

    def fv_residual(self, flagged, solver, RFV):
        f0, f1, f2 = self.fvm()
        g = self.gas
        lib().orc_fv_residual(_p(flagged), flagged.size, _p(self.U), _p(f0), _p(f1), _p(f2),
                              _p(_f(self.basis.weights)), _p(self.J), _p(self.fstar),
                              _p(self.ef_side), _p(self.ef_sign), _p(self.ef_orient), solver,
                              g.gamma, g.R, _p(RFV), self.N)

    def fv_blend(self, solver):
        flagged = np.nonzero(self.alpha > 0.0)[0].astype(np.int64)
        if not flagged.size:
            return
        RFV = np.zeros_like(self.Ut)
        self.fv_residual(flagged, solver, RFV)
        lib().orc_blend(_p(flagged), flagged.size, _p(self.alpha), _p(self.Ut), _p(RFV), self.N)

    def local_dt(self, cfl, cfl_visc):
        g = self.gas
        return lib().orc_local_dt(_p(self.prim), _p(self.Ja), _p(self.J), self.ne, self.N, cfl,
                                  cfl_visc, g.gamma, g.R, g.Pr, g.mu_ref, g.T_ref,
                                  int(g.viscosity_law), int(self.viscous))

    def analysis_partials(self, mu0, g=None):
        """k_analysis_partials (src/testcases.py:190-238): (ne, 9) element rows."""
        gas = self.gas
        out = np.zeros((self.ne, 9), dtype=FT)
        g = self.g if g is None else g
        lib().orc_analysis_partials(_p(self.U), _p(g) if self.viscous else None, _p(self.J),
                                    _p(np.ascontiguousarray(self.basis.weights)), gas.gamma, gas.R,
                                    gas.mu_ref, gas.T_ref, int(gas.viscosity_law),
                                    mu0 if mu0 > 0.0 else 1.0, int(self.viscous), _p(out), self.ne,
                                    self.N)
        return out

    # the time derivative (single-rank order of src/parallel.py:399-517) -------
    def evaluate_rhs(self, t, split=True, surf_solver=RIEMANN_LLF_SPLIT, solver=RIEMANN_LLF,
                     shock=None, source=None):
        self.Ut[...] = 0.0
        self.prolong()
        mins = self.cons_to_prim()
        if self.viscous:
            self.lift()
        bad = self.fill_flux(surf_solver)
        if mins[0] <= 0.0 or mins[1] <= 0.0 or bad >= 0:
            raise ValueError("oracle: inadmissible state")
        self.vol_int(split)
        self.surf_int()
        self.apply_jac()
        if shock is not None:
            self.indicator(shock)
            self.fv_blend(solver)
        if source is not None:
            g = self.gas
            lib().orc_mms_source(_p(self.x), t, _p(self.Ut), self.ne * self.n1 ** 3, source[0],
                                 source[1], g.gamma, g.mu_ref, g.Pr)
        return self.Ut

    def rk_steps(self, nsteps, scheme, cfl, cfl_visc, tend=1e9, t=0.0, **rhs_kw):
        """Reference time loop (src/parallel.py:641-657 + rk_step); returns (t, dts)."""
        work = np.zeros_like(self.U)
        dts = []
        for _ in range(nsteps):
            self.cons_to_prim()
            if not np.isfinite(self.U).all():
                raise FloatingPointError("oracle: non-finite solution")
            dt = self.local_dt(cfl, cfl_visc)
            if t + dt > tend:
                dt = tend - t
            for i in range(scheme.stages):
                Ut = self.evaluate_rhs(t + scheme.c[i] * dt, **rhs_kw)
                lib().orc_lserk(_p(self.U), _p(work), _p(Ut), self.U.size, float(scheme.A[i]),
                                float(scheme.B[i]), dt, int(i == 0))
            t += dt
            dts.append(dt)
        return t, dts
