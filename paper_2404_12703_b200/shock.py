"""FV subcell shock capturing: configuration, subcell metrics, API helpers.

Mirror of ``hexdg.shock`` (reference ``src/shock.py``). The indicator
(:46-110), the first-order FV residual (:113-195) and the convex blend
(:198-210) run on the device fused into the element kernel (see
csrc/kernels.cuh ``volume_kernel``); this module holds the host-side setup
(telescoping subcell interface metrics, computed once) and the API entry
points the reference's tests call.
"""

from dataclasses import dataclass

import numpy as np

from .basis import Basis1D

INDICATOR_HENNEMANN = 0
INDICATOR_CONSTANT = 1

SHARPNESS = float(np.log(1.0 / 1e-4 - 1.0))   # src/shock.py:29


@dataclass(frozen=True)
class ShockConfig:
    enabled: bool = False
    alpha_max: float = 0.5
    alpha_min: float = 1e-3
    indicator: int = INDICATOR_HENNEMANN
    alpha_const: float = 0.0


def modal_threshold(N: int) -> float:
    """T(N) = 0.5 * 10^(-1.8 (N+1)^(1/4)) (src/shock.py:41-43)."""
    return 0.5 * 10.0 ** (-1.8 * (N + 1.0) ** 0.25)


def subcell_interface_metrics(domain):
    """Telescoped subcell interface metrics (src/shock.py:213-257).

    Returns (fvm0, fvm1, fvm2), each (ne, n1, n1, n1+1, 3): the metric at
    interface h of the subcell line with tangential indices ordered as the
    reference ([e, k, j, h] for xi lines, [e, k, i, h] for eta, [e, j, i, h]
    for zeta). Anchored at the element's own face metric so the FV residual
    of a constant state vanishes exactly on curved elements.
    """
    b = domain.basis
    if b.node_type != "LGL":
        raise ValueError("subcell shock capturing requires LGL nodes")
    n1 = b.N + 1
    w, D = b.weights, b.D
    Ja = domain.Ja
    ne = Ja.shape[0]
    out = []
    # (einsum spec, anchor slice, derivative slice along the line axis)
    specs = (("im,ekjmc->ekjic", lambda A: A[:, :, :, 0, :], lambda A, h: A[:, :, :, h, :]),
             ("jm,ekmic->ekjic", lambda A: A[:, :, 0, :, :], lambda A, h: A[:, :, h, :, :]),
             ("km,emjic->ekjic", lambda A: A[:, 0, :, :, :], lambda A, h: A[:, h, :, :, :]))
    for d, (spec, anchor, along) in enumerate(specs):
        dJ = np.einsum(spec, D, Ja[:, d])
        fvm = np.empty((ne, n1, n1, n1 + 1, 3))
        acc = anchor(Ja[:, d]).copy()
        fvm[:, :, :, 0, :] = acc
        for h in range(n1):
            acc = acc + w[h] * along(dJ, h)
            fvm[:, :, :, h + 1, :] = acc
        out.append(np.ascontiguousarray(fvm))
    return tuple(out)


def indicator_alpha(U_elem: np.ndarray, basis: Basis1D, config: ShockConfig,
                    gamma: float = 1.4) -> float:
    """Blending factor of one element's nodal state (k, j, i, 5) (src/shock.py:260-269).

    Evaluated by the device indicator on a one-element domain.
    """
    if config.indicator == INDICATOR_CONSTANT:
        return min(config.alpha_const, config.alpha_max)
    from ._single import single_element_alpha
    return single_element_alpha(np.asarray(U_elem, dtype=np.float64), basis, config, gamma)


def fv_subcell_operator(domain, elem: int, fstar: np.ndarray = None, solver_id: int = 0,
                        fvm=None) -> np.ndarray:
    """First-order FV residual of one element (src/shock.py:272-290), on the device."""
    import ctypes

    from . import _lib
    from .operator import VOL_FVONLY
    d = domain
    dv = d.device
    if fvm is None:
        fvm = subcell_interface_metrics(d)
    dv.set_fvm(fvm)
    dv.upload_state()
    src = d.fstar if fstar is None else fstar
    dv.fstar.copy_(dv.torch.as_tensor(np.ascontiguousarray(src)))
    prm = d.params(split=True, fv_solver=solver_id,
                   shock=ShockConfig(enabled=True, indicator=INDICATOR_CONSTANT, alpha_const=1.0,
                                     alpha_max=1.0))
    out = dv.torch.zeros_like(dv.U)
    _lib.check(dv.lib.hdg_phase_volume(dv.dptr, ctypes.byref(prm), _lib.ptr(dv.U), _lib.ptr(out),
                                       None, 0.0, 0.0, 0.0, 0.0, VOL_FVONLY << 4, dv.sptr()),
               "hdg_phase_volume(FV)")
    return out[elem].cpu().numpy()


def blend(R_DG: np.ndarray, R_FV: np.ndarray, alpha: float) -> np.ndarray:
    """(1 - alpha) R_DG + alpha R_FV with the reference's checks (src/shock.py:293-299)."""
    if not 0.0 <= alpha <= 1.0:
        raise ValueError(f"blending factor {alpha} outside [0, 1]")
    if R_DG.shape != R_FV.shape:
        raise ValueError("operator shapes differ")
    return (1.0 - alpha) * R_DG + alpha * R_FV
