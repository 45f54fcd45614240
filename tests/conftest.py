"""Shared fixtures: golden vectors, domain builders, GPU gating."""

import glob
import os
import sys
import types

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def rhs_golden_names():
    return sorted(os.path.basename(f)[4:-4] for f in glob.glob(os.path.join(GOLDEN, "rhs_*.npz")))


def trajectory_golden_names():
    """Goldens that carry a reference time loop (U_final after len(dts) steps)."""
    out = []
    for n in rhs_golden_names():
        with np.load(os.path.join(GOLDEN, "rhs_" + n + ".npz")) as z:
            if "U_final" in z.files:
                out.append(n)
    return out


def golden_cfg(z):
    from paper_2404_12703_b200.config import RunConfig
    kw = {}
    for k, v in z.items():
        if k.startswith("cfg_"):
            val = v[()]
            if isinstance(val, np.generic):
                val = val.item()
            kw[k[4:]] = val
    return RunConfig(**kw)


def golden_mesh(z):
    from paper_2404_12703_b200 import mesh as mm
    ext = [tuple(r) for r in z["mesh_ext"]]
    m = mm.generate_box_mesh(*[int(n) for n in z["mesh_n"]], ext, tuple(bool(p) for p in z["mesh_per"]))
    if z["mesh_flip_e"].size:
        m = mm.permute_elements(m, z["mesh_flip_e"], [str(k) for k in z["mesh_flip_k"]])
    if float(z["mesh_curve"]):
        m = mm.curve_mesh(m, float(z["mesh_curve"]))
    return m


def solver_ids(cfg):
    split = cfg.operator == "split"
    solver = 1 if cfg.riemann == "hllc" else 0
    return split, solver, (2 if (split and solver == 0) else solver)


def oracle_kwargs(cfg):
    split, solver, surf = solver_ids(cfg)
    shock = None
    if cfg.shockcapture:
        shock = dict(constant=cfg.indicator == "constant", alpha_const=cfg.alphaconst,
                     alpha_max=cfg.alphamax, alpha_min=cfg.alphamin)
    source = (cfg.mmsamplitude, cfg.mmsspeed) if cfg.testcase == "mms" else None
    return dict(split=split, surf_solver=surf, solver=solver, shock=shock, source=source)


def make_worker(cfg, mesh, exact=False):
    """Single-rank product worker (mirror of the reference tests/helpers.py:13-27)."""
    from paper_2404_12703_b200 import testcases
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.mesh import compute_metrics, partition_sfc
    from paper_2404_12703_b200.parallel import RankWorker, SlotLimiter, Transport
    basis = build_basis(cfg.n, cfg.nodetype)
    compute_metrics(mesh, basis)
    parts = partition_sfc(mesh, 1)
    return RankWorker(0, mesh, basis, cfg.gas(), parts[0], np.zeros(mesh.nelem, dtype=np.int64),
                      cfg, Transport(1), SlotLimiter(1), testcases.build_case(cfg), exact=exact)


def oracle_domain(src, cfg):
    import oracle
    from paper_2404_12703_b200.basis import build_basis
    return oracle.OracleDomain(src, build_basis(cfg.n, cfg.nodetype), cfg.gas())


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def normwise(a, b):
    """||a - b||_inf / ||b||_inf over all conserved variables (the parity norm)."""
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def normwise_per_var(a, b):
    """Max over conserved variables of ||a_v - b_v||_inf / ||b_v||_inf (stricter; a
    variable whose RHS nearly cancels, e.g. mass in a Ma 0.1 TGV, sits at 1e-11)."""
    a = a.reshape(-1, 5)
    b = b.reshape(-1, 5)
    den = np.maximum(np.max(np.abs(b), axis=0), 1e-300)
    return float(np.max(np.max(np.abs(a - b), axis=0) / den))


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    from paper_2404_12703_b200 import _lib
    _lib.load()
    import torch
    return torch
