"""Gas model, state types, error types and the array-level physics API.

Mirror of ``hexdg.equations`` (reference ``src/equations.py``). The pointwise
arithmetic (pressure, Sutherland, LLF/HLLC/LLF-split, KEP two-point flux,
viscous flux) lives on the device in ``csrc/physics.cuh``; the array-level
wrappers below (:288-383) validate on the host and evaluate their fluxes through
the device point kernel ``hdg_point_eval``.
"""

from dataclasses import dataclass

import numpy as np

CONST_VISCOSITY = 0          # src/equations.py:14
SUTHERLAND = 1               # src/equations.py:15
N_LIFT = 4                   # lifted set (u, v, w, T), src/equations.py:18

RIEMANN_LLF = 0              # src/equations.py:213-216
RIEMANN_HLLC = 1
RIEMANN_LLF_SPLIT = 2
RIEMANN_SOLVERS = {"llf": RIEMANN_LLF, "hllc": RIEMANN_HLLC}


class AdmissibilityError(ValueError):
    """Non-positive density or pressure reached a flux routine (src/equations.py:21)."""


@dataclass(frozen=True)
class GasProperties:
    """Perfect gas (src/equations.py:25-46); ``viscous`` iff ``mu_ref > 0``."""

    gamma: float = 1.4
    R: float = 287.058
    Pr: float = 0.71
    mu_ref: float = 0.0
    T_ref: float = 273.15
    viscosity_law: int = CONST_VISCOSITY

    def __post_init__(self):
        if self.gamma <= 1.0:
            raise ValueError(f"gamma must exceed 1, got {self.gamma}")
        if self.Pr <= 0.0:
            raise ValueError(f"Prandtl number must be positive, got {self.Pr}")
        if self.mu_ref < 0.0:
            raise ValueError(f"reference viscosity must be >= 0, got {self.mu_ref}")

    @property
    def viscous(self) -> bool:
        return self.mu_ref > 0.0

    def device_table(self) -> np.ndarray:
        """[gamma, R, Pr, mu_ref, T_ref, law] as consumed by hdg_ctx_create."""
        return np.array([self.gamma, self.R, self.Pr, self.mu_ref, self.T_ref,
                         float(self.viscosity_law)], dtype=np.float64)


# ---------------------------------------------------------------------------
# array-level physics API (src/equations.py:288-383). The state conversions and
# the material-law validation are host scalar arithmetic; every flux goes through
# the device point kernels (hdg_point_eval: the same physics.cuh routines as the
# stage kernels, exact kernel set = the reference's operation order).


@dataclass(frozen=True)
class ConservedState:
    rho: float
    mom: tuple
    rhoE: float

    def as_array(self) -> np.ndarray:
        return np.array([self.rho, *self.mom, self.rhoE])


@dataclass(frozen=True)
class PrimitiveState:
    rho: float
    vel: tuple
    p: float
    T: float

    def as_array(self) -> np.ndarray:
        return np.array([self.rho, *self.vel, self.p, self.T])


def _pressure(rho, m0, m1, m2, rhoE, gamma):
    """pt_pressure (src/equations.py:58-63): (gamma-1)(rhoE - 1/2 |m|^2 / rho)."""
    return (gamma - 1.0) * (rhoE - 0.5 * (m0 * m0 + m1 * m1 + m2 * m2) / rho)


def cons_to_prim(U: ConservedState, gas: GasProperties) -> PrimitiveState:
    """Primitive variables (rho, velocity, pressure, temperature) from the state."""
    if U.rho <= 0.0:
        raise AdmissibilityError(f"non-positive density in state {U}")
    vel = tuple(m / U.rho for m in U.mom)
    p = _pressure(U.rho, U.mom[0], U.mom[1], U.mom[2], U.rhoE, gas.gamma)
    if p <= 0.0:
        raise AdmissibilityError(f"non-positive pressure {p} in state {U}")
    return PrimitiveState(rho=U.rho, vel=vel, p=p, T=p / (U.rho * gas.R))


def prim_to_cons(P: PrimitiveState, gas: GasProperties) -> ConservedState:
    if P.rho <= 0.0 or P.p <= 0.0:
        raise AdmissibilityError(f"non-positive density or pressure in state {P}")
    mom = tuple(P.rho * v for v in P.vel)
    rhoE = P.p / (gas.gamma - 1.0) + 0.5 * P.rho * sum(v * v for v in P.vel)
    return ConservedState(rho=P.rho, mom=mom, rhoE=rhoE)


POINT_EULER_FLUX_DIR, POINT_VISCOUS_FLUX_DIR, POINT_RIEMANN = 0, 1, 2
POINT_SPLIT_KEP, POINT_VISCOSITY, POINT_CONDUCTIVITY = 3, 4, 5
_POINT_OUT = {0: 5, 1: 5, 2: 5, 3: 5, 4: 1, 5: 1}


def point_eval(op: int, rows, gas: GasProperties, solver: int = RIEMANN_LLF) -> np.ndarray:
    """Evaluate a device point routine for every row of ``rows`` (hdg_point_eval,
    the exact kernel set): (n, width_in) -> (n, width_out)."""
    import ctypes

    from . import _lib
    torch = _lib.require_cuda()
    lib = _lib.load()
    x = np.ascontiguousarray(np.atleast_2d(np.asarray(rows, dtype=np.float64)))
    dev = torch.device("cuda", torch.cuda.current_device())
    xin = torch.as_tensor(x, device=dev)
    out = torch.zeros((x.shape[0], _POINT_OUT[op]), dtype=torch.float64, device=dev)
    p = _lib.HdgParams()
    p.gamma, p.R, p.Pr, p.mu_ref, p.T_ref = gas.gamma, gas.R, gas.Pr, gas.mu_ref, gas.T_ref
    p.law = int(gas.viscosity_law)
    p.exact = 1
    _lib.check(lib.hdg_point_eval(ctypes.byref(p), int(op), int(solver), x.shape[0],
                                  _lib.ptr(xin), _lib.ptr(out), _lib.stream_ptr()),
               "hdg_point_eval")
    return out.cpu().numpy()


def viscosity(T: float, gas: GasProperties) -> float:
    if T <= 0.0:
        raise AdmissibilityError(f"non-positive temperature {T}")
    return float(point_eval(POINT_VISCOSITY, [[T]], gas)[0, 0])


def thermal_conductivity(mu: float, gas: GasProperties) -> float:
    if mu < 0.0:
        raise AdmissibilityError(f"negative viscosity {mu}")
    return float(point_eval(POINT_CONDUCTIVITY, [[mu]], gas)[0, 0])


def euler_flux(P: PrimitiveState, U: ConservedState) -> np.ndarray:
    """Physical convective fluxes, one 5-vector per Cartesian direction; shape (3, 5)."""
    rows = [[P.rho, P.vel[0], P.vel[1], P.vel[2], P.p, U.rhoE, *n] for n in np.eye(3)]
    return point_eval(POINT_EULER_FLUX_DIR, rows, GasProperties())


def viscous_flux(P: PrimitiveState, gradP: np.ndarray, gas: GasProperties) -> np.ndarray:
    """Viscous fluxes from the (3, 4) gradient of (u, v, w, T); shape (3, 5)."""
    g = np.asarray(gradP, dtype=np.float64)
    if g.shape != (3, N_LIFT):
        raise ValueError(f"gradient must have shape (3, {N_LIFT}), got {g.shape}")
    viscosity(P.T, gas)   # the reference's admissibility checks
    rows = [[P.vel[0], P.vel[1], P.vel[2], P.T, *g.ravel(), *n] for n in np.eye(3)]
    return point_eval(POINT_VISCOUS_FLUX_DIR, rows, gas)


def riemann_flux(PL: PrimitiveState, PR: PrimitiveState, n: np.ndarray,
                 gas: GasProperties, solver: str = "llf") -> np.ndarray:
    """Common interface flux f*(UL, UR, n) for a unit normal."""
    n = np.asarray(n, dtype=np.float64)
    if abs(np.linalg.norm(n) - 1.0) > 1e-12:
        raise ValueError(f"normal must have unit length, got |n|={np.linalg.norm(n)}")
    for P in (PL, PR):
        if P.rho <= 0.0 or P.p <= 0.0:
            raise AdmissibilityError(f"inadmissible interface state {P}")
    UL, UR = prim_to_cons(PL, gas), prim_to_cons(PR, gas)
    row = [PL.rho, *PL.vel, PL.p, UL.rhoE, PR.rho, *PR.vel, PR.p, UR.rhoE, *n]
    return point_eval(POINT_RIEMANN, [row], gas, RIEMANN_SOLVERS[solver])[0]


def split_flux_twopoint(PL: PrimitiveState, PR: PrimitiveState,
                        metric: np.ndarray, gas: GasProperties) -> np.ndarray:
    """Symmetric two-point volume flux in the direction of a metric vector."""
    UL, UR = prim_to_cons(PL, gas), prim_to_cons(PR, gas)
    m = np.asarray(metric, dtype=np.float64)
    row = [PL.rho, *PL.vel, PL.p, (UL.rhoE + PL.p) / PL.rho,
           PR.rho, *PR.vel, PR.p, (UR.rhoE + PR.p) / PR.rho, *m]
    return point_eval(POINT_SPLIT_KEP, [row], gas)[0]


def br1_lifting_flux(PL: PrimitiveState, PR: PrimitiveState) -> np.ndarray:
    """Central (arithmetic mean) trace of the lifted variable set (u, v, w, T)."""
    vL = np.array([*PL.vel, PL.T])
    vR = np.array([*PR.vel, PR.T])
    return 0.5 * (vL + vR)
