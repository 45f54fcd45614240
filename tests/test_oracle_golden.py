"""The oracle is pinned: bit-identical to the reference on every golden vector.

Golden vectors were produced by the reference package itself
(tests/golden/make_golden.py). CPU only.
"""

import types

import numpy as np
import pytest

from conftest import (golden, golden_cfg, oracle_domain, oracle_kwargs, rhs_golden_names,
                      trajectory_golden_names)


@pytest.mark.parametrize("name", rhs_golden_names())
def test_oracle_rhs_bitwise(name):
    z = golden("rhs_" + name)
    cfg = golden_cfg(z)
    od = oracle_domain(types.SimpleNamespace(**z), cfg)
    od.U[...] = z["U0"]
    od.bc_states[...] = z["bc_states"]
    Ut = od.evaluate_rhs(float(z["t"]), **oracle_kwargs(cfg))
    assert np.array_equal(Ut, z["Ut"])
    assert np.array_equal(od.fstar, z["fstar"])
    if "prim" in z:
        assert np.array_equal(od.prim, z["prim"])
    if "g" in z:
        assert np.array_equal(od.g, z["g"])
        assert np.array_equal(od.gL, z["gL"])
        assert np.array_equal(od.vstar, z["vstar"])
        assert np.array_equal(od.Fvis, z["Fvis"])
    if cfg.shockcapture:
        assert np.array_equal(od.alpha, z["alpha"])
        f = od.fvm()
        for d in range(3):
            assert np.array_equal(f[d], z[f"fvm{d}"])
    assert od.local_dt(cfg.cfl, cfg.cflvisc) == float(z["dt"])


@pytest.mark.parametrize("name", trajectory_golden_names())
def test_oracle_trajectory_bitwise(name):
    from paper_2404_12703_b200.timedisc import get_scheme
    z = golden("rhs_" + name)
    cfg = golden_cfg(z)
    od = oracle_domain(types.SimpleNamespace(**z), cfg)
    od.U[...] = z["U0"]
    t, dts = od.rk_steps(len(z["dts"]), get_scheme(cfg.rkscheme), cfg.cfl, cfg.cflvisc,
                         **oracle_kwargs(cfg))
    assert np.array_equal(np.array(dts), z["dts"])
    assert t == float(z["t_final"])
    assert np.array_equal(od.U, z["U_final"])


def test_oracle_hennemann_flags_some_elements():
    z = golden("rhs_euler_hennemann_n5")
    assert 0 < int(np.sum(z["alpha"] > 0)) < z["alpha"].size


def test_extended_oracle_measures_the_references_own_error():
    """The long double oracle (the parity tests' yardstick) agrees with the double
    oracle to double precision on a well-conditioned RHS, and shows the reference's
    own floating-point error on the ill-conditioned unperturbed Ma 0.1 vortex (its Ut
    is ~1e-4 of the pressure terms it is summed from)."""
    import oracle
    from paper_2404_12703_b200.basis import build_basis
    errs = {}
    for name in ("ns_split_n3", "tgv_ns_split_n7"):
        z = golden("rhs_" + name)
        cfg = golden_cfg(z)
        oracle.extended(True)
        try:
            od = oracle.OracleDomain(types.SimpleNamespace(**z), build_basis(cfg.n, cfg.nodetype),
                                     cfg.gas())
            od.U[...] = z["U0"]
            od.bc_states[...] = z["bc_states"]
            hp = np.array(od.evaluate_rhs(float(z["t"]), **oracle_kwargs(cfg)), dtype=np.longdouble)
        finally:
            oracle.extended(False)
        errs[name] = float(np.max(np.abs(z["Ut"] - hp)) / np.max(np.abs(hp)))
    assert errs["ns_split_n3"] < 1e-14
    assert 1e-13 < errs["tgv_ns_split_n7"] < 1e-11, errs
