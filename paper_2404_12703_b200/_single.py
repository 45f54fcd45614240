"""Single-element device evaluations used by API helpers (shock.indicator_alpha)."""

import ctypes

import numpy as np

from . import _lib
from .basis import pack_basis


def single_element_alpha(U_elem, basis, config, gamma):
    """Run the device modal indicator (src/shock.py:46-110) on one element."""
    from .shock import SHARPNESS, modal_threshold
    torch = _lib.require_cuda()
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    n1 = basis.N + 1
    U = torch.as_tensor(np.ascontiguousarray(U_elem.reshape(1, n1, n1, n1, 5)), device=dev)
    b = torch.as_tensor(pack_basis(basis), device=dev)
    alpha = torch.zeros(1, dtype=torch.float64, device=dev)
    status = torch.zeros(8, dtype=torch.int32, device=dev)
    out = torch.zeros_like(U)
    D = _lib.HdgDomain()
    D.N, D.node_type, D.ne, D.ns = basis.N, 0, 1, 0
    D.basis, D.alpha, D.status = _lib.ptr(b), _lib.ptr(alpha), _lib.ptr(status)
    P = _lib.HdgParams()
    P.gamma = gamma
    P.split, P.shock, P.indicator = 1, 1, 0
    thr = modal_threshold(basis.N)
    P.alpha_max, P.alpha_min = config.alpha_max, config.alpha_min
    P.ind_threshold, P.ind_slope = thr, -SHARPNESS / thr
    P.exact = 1
    _lib.check(lib.hdg_phase_volume(ctypes.byref(D), ctypes.byref(P), _lib.ptr(U), _lib.ptr(out),
                                    None, 0.0, 0.0, 0.0, 0.0, 32 << 4, _lib.stream_ptr()),
               "hdg_phase_volume(indicator)")
    return float(alpha.cpu().numpy()[0])
