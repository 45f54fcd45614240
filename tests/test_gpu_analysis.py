"""Device analysis partials and the time loop with analysis (RankWorker.analyze,
src/parallel.py:606-665) vs the reference's own outputs (tests/golden)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _domain(n, curve, mu_ref, m=2):
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.equations import GasProperties
    from paper_2404_12703_b200.mesh import compute_metrics, curve_mesh, generate_box_mesh
    from paper_2404_12703_b200.operator import Domain
    two_pi = 2 * np.pi
    mesh = generate_box_mesh(m, m, m, [(0.0, two_pi)] * 3, (True,) * 3)
    if curve:
        mesh = curve_mesh(mesh, curve)
    basis = build_basis(n)
    compute_metrics(mesh, basis)
    return Domain(mesh, basis, GasProperties(mu_ref=mu_ref))


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
def test_device_analysis_partials_match_reference(gpu, exact):
    from paper_2404_12703_b200.testcases import analysis_partials
    z = golden("analysis_partials")
    d = _domain(4, 0.05, 1.0 / 1600.0)
    d.exact = exact
    d.U[...] = z["ns_U"]
    d.g[...] = z["ns_g"]
    rows = analysis_partials(d, float(z["ns_mu0"]))
    if exact:
        assert np.array_equal(rows, z["ns_partials"])
    else:
        assert np.max(np.abs(rows - z["ns_partials"])) <= 1e-13 * np.max(np.abs(z["ns_partials"]))
    d = _domain(3, 0.0, 0.0)
    d.exact = exact
    d.U[...] = z["eu_U"]
    rows = analysis_partials(d, 0.0)
    if exact:
        assert np.array_equal(rows, z["eu_partials"])
    else:
        assert np.max(np.abs(rows - z["eu_partials"])) <= 1e-13 * np.max(np.abs(z["eu_partials"]))


@pytest.mark.parametrize("viscous", [True, False], ids=["ns", "euler"])
def test_run_series_bitwise_equal_reference(gpu, monkeypatch, viscous):
    """run_distributed with analyzeinterval=2: the analysis rows (t, E_k, eps_S,
    eps_D, dt, integrals) and the final field equal the reference's bit for bit."""
    from paper_2404_12703_b200.config import RunConfig
    from paper_2404_12703_b200.parallel import run_distributed
    monkeypatch.setenv("HEXDG_EXACT", "1")
    z = golden("run_series")
    tag = "ns" if viscous else "eu"
    two_pi = 2 * np.pi
    cfg = RunConfig(testcase="tgv", n=3, mach=0.1, muref=(1.0 / 1600.0) if viscous else 0.0,
                    meshx=3, meshy=3, meshz=3, maxsteps=5, analyzeinterval=2, tend=1e9,
                    x0=0.0, x1=two_pi, y0=0.0, y1=two_pi, z0=0.0, z1=two_pi)
    seen = []
    res = run_distributed(cfg, on_analyze=lambda t, q, U, a: seen.append((t, U.shape, a.shape)))
    cols = [str(c) for c in z["columns"]]
    ref = z[tag + "_series"]
    assert len(res.series) == ref.shape[0] == len(seen) == 4
    for row, r in zip(res.series, ref):
        for c in cols:
            assert row.get(c, 0.0) == r[cols.index(c)], (c, row.get(c), r[cols.index(c)])
    assert np.array_equal(res.U, z[tag + "_U"])
    assert res.t == float(z[tag + "_t"])
    # the reference's row layout for the callback (src/parallel.py:621-623)
    ne = res.U.shape[0]
    assert seen[0][1] == (ne, res.U[0].size) and seen[0][2] == (ne, 1)


def test_tgv_version1_kinetic_energy(gpu):
    """tests/test_testcases.py:130-135 on the device analysis path."""
    from paper_2404_12703_b200.testcases import (TGVSetup, analysis_partials,
                                                 reduce_tgv_quantities, tgv_init)
    setup = TGVSetup(mach=0.1, reynolds=1600.0, version=1)
    d = _domain(5, 0.0, 0.0, m=4)   # tgv_domain(setup), tests/test_testcases.py:111-117
    d.U[...] = tgv_init(setup, d.x, d.gas)
    q = reduce_tgv_quantities(analysis_partials(d, setup.mu0()), setup)
    assert abs(q["E_k"] - 0.125) < 1e-10


def test_tgv_initial_field_nearly_divergence_free(gpu):
    """tests/test_testcases.py:171-181."""
    from paper_2404_12703_b200.config import RunConfig
    from paper_2404_12703_b200.parallel import run_distributed
    cfg = RunConfig(testcase="tgv", n=7, meshx=4, meshy=4, meshz=4, x0=0.0, x1=2 * np.pi,
                    y0=0.0, y1=2 * np.pi, z0=0.0, z1=2 * np.pi, mach=0.1, reynolds=1600.0,
                    muref=1.0 / 1600.0, tgvversion=2, operator="split", nodetype="LGL",
                    tend=1e9, maxsteps=1, analyzeinterval=0)
    res = run_distributed(cfg)
    row = res.series[0]
    assert row["eps_D"] < 1e-4 * row["eps_S"]


@pytest.mark.parametrize("shock", [False, True], ids=["ns", "ns_fv"])
def test_restart_from_snapshot_bitwise(gpu, tmp_path, shock):
    """Resume (new; the reference has none): K steps -> HDGF snapshot -> restartfile
    run of K more steps equals the uninterrupted 2K-step run bit for bit (U and t)."""
    from paper_2404_12703_b200.config import RunConfig
    from paper_2404_12703_b200.io import write_snapshot
    from paper_2404_12703_b200.parallel import run_distributed
    two_pi = 2 * np.pi
    kw = dict(testcase="tgv", n=3, mach=0.3, muref=1.0 / 400.0, meshx=3, meshy=3, meshz=3,
              tend=1e9, analyzeinterval=0, x0=0.0, x1=two_pi, y0=0.0, y1=two_pi, z0=0.0,
              z1=two_pi)
    if shock:
        kw.update(shockcapture=True, indicator="constant", alphaconst=0.3)
    full = run_distributed(RunConfig(maxsteps=6, **kw))
    half = run_distributed(RunConfig(maxsteps=3, **kw))
    snap = tmp_path / "half.hdgf"
    write_snapshot(snap, half.U, half.t, half.alpha)
    resumed = run_distributed(RunConfig(maxsteps=3, restartfile=str(snap), **kw))
    assert resumed.t == full.t
    assert np.array_equal(resumed.U, full.U)
    # the stitched series: no duplicated row at the snapshot time
    kw2 = dict(kw, analyzeinterval=1)
    full_s = run_distributed(RunConfig(maxsteps=6, **kw2)).series
    half_s = run_distributed(RunConfig(maxsteps=3, **kw2)).series
    res_s = run_distributed(RunConfig(maxsteps=3, restartfile=str(snap), **kw2)).series
    stitched = half_s + res_s
    assert [r["t"] for r in stitched] == [r["t"] for r in full_s]
    for a, b in zip(stitched, full_s):
        assert a["E_k"] == b["E_k"]
