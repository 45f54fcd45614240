"""Every degree the library instantiates (N = 1..7) through the production RHS path,
in the configurations the dispatch distinguishes -- LGL split Navier-Stokes / Euler, each
with and without FV-subcell blending, GL standard Navier-Stokes with HLLC, LGL standard
Euler -- on a small curved, randomly flipped periodic mesh, against the oracle:
the exact set bit for bit, the fast set within the parity tolerance. Catches layout
and alignment faults of degree-specific shared-memory maps (odd n1 / n3) that the
configuration-specific tests do not reach."""

import numpy as np
import pytest

from conftest import make_worker, normwise, oracle_domain, oracle_kwargs

pytestmark = pytest.mark.gpu

CASES = {
    "ns-split": dict(muref=1.0 / 1600.0),
    "euler-split": dict(muref=0.0),
    "ns-split-fv": dict(muref=1.0 / 1600.0, shockcapture=True, indicator="constant",
                        alphaconst=0.3),
    "ns-gl-standard-hllc": dict(muref=1.0 / 1600.0, nodetype="GL", operator="standard",
                                riemann="hllc"),
    "euler-split-fv": dict(muref=0.0, shockcapture=True, indicator="constant", alphaconst=0.3),
    "euler-lgl-standard": dict(muref=0.0, operator="standard"),
}


def _case(n, name, exact):
    from paper_2404_12703_b200 import mesh as mm
    from paper_2404_12703_b200.config import RunConfig
    two_pi = 2 * np.pi
    cfg = RunConfig(testcase="tgv", n=n, mach=0.5, meshx=3, meshy=3, meshz=3, x0=0.0,
                    x1=two_pi, y0=0.0, y1=two_pi, z0=0.0, z1=two_pi, tend=1e9,
                    **CASES[name])
    m = mm.curve_mesh(mm.random_flips(mm.generate_box_mesh(3, 3, 3, [(0.0, two_pi)] * 3,
                                                           (True,) * 3), seed=n), 0.03)
    return cfg, make_worker(cfg, m, exact=exact)


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("n", list(range(1, 8)))
def test_degree_configuration_matrix(gpu, n, name, exact):
    import torch
    cfg, w = _case(n, name, exact)
    d = w.domain
    od = oracle_domain(d, cfg)
    od.U[...] = d.U
    ref = od.evaluate_rhs(0.0, **oracle_kwargs(cfg)).copy()
    w._prepare()
    dv = d.device
    dv.upload_state()
    Ut = torch.empty_like(dv.U)
    w.rhs_device(dv.U, Ut, 0.0)
    Ut = Ut.cpu().numpy()
    assert np.isfinite(Ut).all()
    if exact:
        assert np.array_equal(Ut, ref), normwise(Ut, ref)
    else:
        assert normwise(Ut, ref) <= 1e-12, normwise(Ut, ref)
