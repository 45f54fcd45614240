"""Gas model constants and the error types of the physics layer.

Host-side mirror of ``hexdg.equations`` (reference ``src/equations.py``). The
pointwise arithmetic itself (pressure, Sutherland, LLF/HLLC/LLF-split, KEP
two-point flux, viscous flux) lives on the device in ``csrc/physics.cuh``;
this module only carries the frozen gas description that is uploaded to the
device and the solver ids / exception types the Python API exposes.
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
