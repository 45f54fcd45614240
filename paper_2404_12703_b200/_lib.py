"""ctypes binding of ``csrc/libhexdg_b200.so`` (the C ABI in include/hexdg_b200.h).

There is no CPU fallback: importing the operator on a machine without the
built library or without a CUDA device raises :class:`HexdgNativeError` at the
first device call. Device memory and streams come from PyTorch (plumbing
only); every compute call goes through this library.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HEXDG_B200_LIB overrides the in-tree library (A/B builds of the same ABI)
LIB_PATH = os.environ.get("HEXDG_B200_LIB") or os.path.join(_HERE, "csrc", "libhexdg_b200.so")


class HexdgNativeError(RuntimeError):
    """The CUDA library is missing, failed to load, or a call returned an error."""


c_dp = ctypes.c_void_p


class HdgDomain(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int32), ("node_type", ctypes.c_int32),
        ("ne", ctypes.c_int32), ("ns", ctypes.c_int32),
        ("basis", c_dp), ("Ja", c_dp), ("J", c_dp), ("invJ", c_dp), ("nvec", c_dp),
        ("ssurf", c_dp), ("x", c_dp), ("ef_info", c_dp), ("side_info", c_dp),
        ("bc_states", c_dp), ("fvm0", c_dp), ("fvm1", c_dp), ("fvm2", c_dp),
        ("UL", c_dp), ("UR", c_dp), ("fstar", c_dp), ("Fvis", c_dp), ("fvface", c_dp),
        ("g", c_dp), ("gL", c_dp), ("gR", c_dp), ("vstar", c_dp), ("alpha", c_dp),
        ("status", c_dp), ("dt_bits", c_dp), ("vol", c_dp),
        ("rfv", c_dp), ("fv_list", c_dp), ("fv_count", c_dp), ("work", c_dp),
    ]


class HdgParams(ctypes.Structure):
    _fields_ = [
        ("gamma", ctypes.c_double), ("R", ctypes.c_double), ("Pr", ctypes.c_double),
        ("mu_ref", ctypes.c_double), ("T_ref", ctypes.c_double),
        ("law", ctypes.c_int32), ("viscous", ctypes.c_int32), ("split", ctypes.c_int32),
        ("surf_solver", ctypes.c_int32), ("fv_solver", ctypes.c_int32),
        ("shock", ctypes.c_int32), ("indicator", ctypes.c_int32),
        ("alpha_max", ctypes.c_double), ("alpha_min", ctypes.c_double),
        ("alpha_const", ctypes.c_double), ("ind_threshold", ctypes.c_double),
        ("ind_slope", ctypes.c_double), ("source", ctypes.c_int32),
        ("mms_A", ctypes.c_double), ("mms_a", ctypes.c_double),
        ("exact", ctypes.c_int32), ("pad", ctypes.c_int32),
        ("cfl", ctypes.c_double), ("cfl_visc", ctypes.c_double),
    ]


class HdgGate(ctypes.Structure):
    _fields_ = [("flags", c_dp), ("idx", c_dp), ("n", ctypes.c_int32), ("pos", ctypes.c_int32),
                ("epoch", c_dp)]


STATUS_BAD_PRIM, STATUS_BAD_SIDE, STATUS_NONFINITE, STATUS_PEER_TIMEOUT = 0, 1, 2, 3
MODE_STORE_UT, MODE_LSERK, MODE_LSERK_FIRST = 0, 1, 2

_SIGS = {
    "hdg_abi_version": (ctypes.c_int, []),
    "hdg_last_error": (ctypes.c_char_p, []),
    "hdg_sizeof_domain": (ctypes.c_int64, []),
    "hdg_sizeof_params": (ctypes.c_int64, []),
    "hdg_launch_count": (ctypes.c_int64, []),
    "hdg_check_domain": (ctypes.c_int, [c_dp, c_dp]),
    "hdg_rhs": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, ctypes.c_double, c_dp, ctypes.c_int32, c_dp]),
    "hdg_stage": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, c_dp, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_int, c_dp, ctypes.c_int32, c_dp]),
    "hdg_phase_lift": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp]),
    "hdg_phase_elem": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp]),
    "hdg_phase_elem_list": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, ctypes.c_int32, ctypes.c_int,
                                           c_dp]),
    "hdg_phase_update_list": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, c_dp, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_int, c_dp, ctypes.c_int32, ctypes.c_int,
                                             c_dp]),
    "hdg_phase_update": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, c_dp, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_int, c_dp]),
    "hdg_phase_flux": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, ctypes.c_int32, ctypes.c_int32, c_dp]),
    "hdg_phase_volume": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, c_dp, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_int, c_dp]),
    "hdg_cons_to_prim": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, c_dp]),
    "hdg_prolong": (ctypes.c_int, [c_dp, c_dp, c_dp, ctypes.c_int32, c_dp]),
    "hdg_apply_bc_traces": (ctypes.c_int, [c_dp, c_dp, ctypes.c_int32, c_dp]),
    "hdg_fill_flux_traces": (ctypes.c_int, [c_dp, c_dp, c_dp, ctypes.c_int32, ctypes.c_int32, c_dp]),
    "hdg_surf_int": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp]),
    "hdg_apply_jac": (ctypes.c_int, [c_dp, c_dp, c_dp]),
    "hdg_local_dt": (ctypes.c_int, [c_dp, c_dp, c_dp, ctypes.c_double, ctypes.c_double, c_dp]),
    "hdg_dt_finalize": (ctypes.c_int, [c_dp, c_dp, ctypes.c_double, c_dp]),
    "hdg_time_advance": (ctypes.c_int, [c_dp, c_dp]),
    "hdg_analysis_partials": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, ctypes.c_double, c_dp, c_dp]),
    "hdg_lserk_update": (ctypes.c_int, [c_dp, c_dp, c_dp, ctypes.c_int64, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_int, c_dp]),
    "hdg_pack": (ctypes.c_int, [c_dp, c_dp, ctypes.c_int32, ctypes.c_int32, c_dp, c_dp]),
    "hdg_unpack": (ctypes.c_int, [c_dp, c_dp, ctypes.c_int32, ctypes.c_int32, c_dp, c_dp]),
    "hdg_pack_traces": (ctypes.c_int, [c_dp, c_dp, c_dp, ctypes.c_int32, c_dp, c_dp]),
    "hdg_peer_send_traces": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, c_dp, ctypes.c_int32, c_dp,
                                            c_dp, ctypes.c_int32, c_dp, c_dp, c_dp]),
    "hdg_peer_send_rows": (ctypes.c_int, [c_dp, ctypes.c_int32, c_dp, c_dp, c_dp, ctypes.c_int32,
                                          c_dp, c_dp, ctypes.c_int32, c_dp, c_dp, c_dp]),
    "hdg_peer_wait": (ctypes.c_int, [c_dp, c_dp, ctypes.c_int32, c_dp, c_dp, c_dp]),
    "hdg_peer_allreduce_dt": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, c_dp, ctypes.c_int32,
                                             ctypes.c_int32, c_dp, c_dp]),
    "hdg_ipc_export": (ctypes.c_int, [c_dp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)]),
    "hdg_ipc_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(c_dp)]),
    "hdg_phase_elem_gated": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, ctypes.c_int32, ctypes.c_int,
                                            c_dp, c_dp]),
    "hdg_phase_flux_gated": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, ctypes.c_int32, ctypes.c_int32,
                                            c_dp, c_dp]),
    "hdg_phase_update_gated": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp, c_dp, ctypes.c_double,
                                              ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                              ctypes.c_int, c_dp, ctypes.c_int32, ctypes.c_int,
                                              c_dp, c_dp]),
    "hdg_ipc_close": (ctypes.c_int, [c_dp]),
    "hdg_point_eval": (ctypes.c_int, [c_dp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_dp,
                                      c_dp, c_dp]),
    "hdg_mms_source": (ctypes.c_int, [c_dp, ctypes.c_int32, c_dp, ctypes.c_double, c_dp, c_dp]),
    "hdg_lift_fill": (ctypes.c_int, [c_dp, c_dp, c_dp, ctypes.c_int32, c_dp]),
    "hdg_lift_volume": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp]),
    "hdg_lift_finish": (ctypes.c_int, [c_dp, c_dp, c_dp, c_dp]),
    "hdg_debug_phase_cycles": (ctypes.c_int, [ctypes.c_int, c_dp]),
}

EXPORTED = tuple(_SIGS)
ABI_VERSION = 2            # include/hexdg_b200.h HDG_ABI_VERSION
STAGE_NEXT_DT = 2          # hdg_stage first-bit: fold the next step dt into the stage
_lib = None


def load(path: str = LIB_PATH):
    """Load the library once; raise HexdgNativeError if it is absent or stale."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise HexdgNativeError(
            f"{path} not built; run `python -m paper_2404_12703_b200.build` (no CPU fallback)")
    try:
        lib = ctypes.CDLL(path)
    except OSError as exc:
        raise HexdgNativeError(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.hdg_abi_version() != ABI_VERSION:
        raise HexdgNativeError("libhexdg_b200 ABI version mismatch")
    if (lib.hdg_sizeof_domain() != ctypes.sizeof(HdgDomain)
            or lib.hdg_sizeof_params() != ctypes.sizeof(HdgParams)):
        raise HexdgNativeError("hdg_domain / hdg_params layout differs from the ctypes binding")
    _lib = lib
    return lib


def check(rc: int, what: str):
    if rc != 0:
        msg = _lib.hdg_last_error().decode(errors="replace") if _lib else ""
        raise HexdgNativeError(f"{what} failed (rc={rc}): {msg}")


def ptr(t):
    """Device pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise HexdgNativeError("no CUDA device visible: the hexdg_b200 hot path has no CPU fallback")
    load()
    return torch


def require_device_f64(t, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
            and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous CUDA float64 tensor")


def lserk_update(U, dU, Ut, A, B, dt, first=False, stream=None):
    lib = load()
    check(lib.hdg_lserk_update(ptr(U), ptr(dU), ptr(Ut), U.numel(), A, B, dt, int(first),
                               stream_ptr(stream)), "hdg_lserk_update")
