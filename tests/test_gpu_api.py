"""The reference's remaining Python surface through the device kernels:
raw k_surf_int, the split lifting calls, the array-level physics API, the MMS
source, rk_step on host arrays -- each against the reference's own values."""

import types

import numpy as np
import pytest

from conftest import golden, golden_cfg, golden_mesh, make_worker

pytestmark = pytest.mark.gpu


def test_k_surf_int_pencil_and_paper(gpu):
    """tests/test_operator.py:99-118 with the raw kernel call: a unit flux on one
    side gives -1/w0 ... at the replica's face nodes and +1/wN at the primary's."""
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.equations import GasProperties
    from paper_2404_12703_b200.mesh import compute_metrics, generate_box_mesh
    from paper_2404_12703_b200.operator import Domain, k_surf_int
    b = build_basis(3, "LGL")
    m = generate_box_mesh(2, 1, 1, [(0.0, 2.0), (0.0, 1.0), (0.0, 1.0)], (True, True, True))
    compute_metrics(m, b)
    d = Domain(m, b, GasProperties())
    fstar = np.zeros_like(d.fstar)
    s = int(d.ef_side[0, 1])                 # element 0, xi+ side (primary)
    fstar[s, :, :, 0] = 1.0
    Ut = np.zeros_like(d.Ut)
    k_surf_int(fstar, d.ef_side, d.ef_sign, d.ef_orient, b.lhat_minus, b.lhat_plus, Ut)
    assert np.allclose(Ut[0, :, :, 3, 0], b.lhat_plus[3])
    nb = int(m.side_elem_r[d.side_global[s]]) - d.lo
    assert np.allclose(Ut[nb, :, :, 0, 0], -b.lhat_minus[0])
    assert np.count_nonzero(Ut[..., 0]) == 2 * 16


def test_k_surf_int_gather_equals_oracle_bitwise(gpu):
    """Criterion 8 (tests/test_acceptance.py:187-202) and bitwise vs the oracle's
    k_surf_int restatement on the all-orientation mesh."""
    import oracle
    from paper_2404_12703_b200.operator import k_surf_int
    z = golden("rhs_ns_split_n3")
    cfg = golden_cfg(z)
    w = make_worker(cfg, golden_mesh(z), exact=True)
    d = w.domain
    b = d.basis
    assert {int(c) for c in np.unique(d.ef_orient)} == {0, 1, 2, 3}
    rng = np.random.default_rng(2024)
    fstar = 0.01 * rng.standard_normal(d.fstar.shape)
    Ut = np.zeros_like(d.Ut)
    k_surf_int(fstar, d.ef_side, d.ef_sign, d.ef_orient, b.lhat_minus, b.lhat_plus, Ut)
    od = oracle.OracleDomain(d, b, cfg.gas())
    ref = od.surf_int(fstar=fstar, Ut=np.zeros_like(d.Ut))
    assert np.array_equal(Ut, ref)


@pytest.mark.parametrize("name", ["ns_split_n3", "ns_std_gl_walls_n3", "tgv_ns_split_n7"])
def test_split_lifting_calls_match_reference(gpu, name):
    """Domain.prolong -> lift_fill -> lift_volume -> lift_finish, the reference's call
    sequence (src/parallel.py:449-499), bit-identical vstar / g / Fvis."""
    z = golden("rhs_" + name)
    cfg = golden_cfg(z)
    w = make_worker(cfg, golden_mesh(z), exact=True)
    d = w.domain
    d.U[...] = z["U0"]
    d.bc_states[...] = z["bc_states"]
    d.prolong(False)
    assert np.array_equal(d.UL, z["UL"]) and np.array_equal(d.UR, z["UR"])
    d.lift_fill(d.sides_inner)
    assert np.array_equal(d.vstar, z["vstar"])
    d.lift_volume()
    d.lift_finish()
    assert np.array_equal(d.g, z["g"])
    assert np.array_equal(d.Fvis, z["Fvis"])


def _gas(row):
    from paper_2404_12703_b200.equations import GasProperties
    return GasProperties(gamma=row[0], R=row[1], Pr=row[2], mu_ref=row[3], T_ref=row[4],
                         viscosity_law=int(row[5]))


@pytest.mark.parametrize("tag", ["const", "suth"])
def test_array_physics_api_bitwise(gpu, tag):
    """equations.riemann_flux / split_flux_twopoint / euler_flux / viscous_flux /
    viscosity / thermal_conductivity / prim_to_cons vs the reference's values."""
    from paper_2404_12703_b200 import equations as eq
    z = golden("physics_points")
    gas = _gas(z[f"{tag}_gas"])
    # Python floats, as the reference's callers pass them: Python 3.12's sum() over exact
    # floats (prim_to_cons' kinetic energy) is compensated, over numpy scalars it is not
    P = [eq.PrimitiveState(rho=float(r[0]), vel=tuple(float(v) for v in r[1:4]), p=float(r[4]),
                           T=float(r[5])) for r in z[f"{tag}_prims"]]
    n = z[f"{tag}_normals"].shape[0]
    for solver in ("llf", "hllc"):
        got = np.array([eq.riemann_flux(P[2 * k], P[2 * k + 1], z[f"{tag}_normals"][k], gas, solver)
                        for k in range(n)])
        assert np.array_equal(got, z[f"{tag}_riemann_{solver}"]), solver
    got = np.array([eq.split_flux_twopoint(P[2 * k], P[2 * k + 1], z[f"{tag}_metrics"][k], gas)
                    for k in range(n)])
    assert np.array_equal(got, z[f"{tag}_kep"])
    got = np.array([eq.euler_flux(P[k], eq.prim_to_cons(P[k], gas)) for k in range(n)])
    assert np.array_equal(got, z[f"{tag}_euler"])
    got = np.array([eq.viscous_flux(P[k], z[f"{tag}_grads"][k], gas) for k in range(n)])
    assert np.array_equal(got, z[f"{tag}_viscous"])
    mu = np.array([eq.viscosity(P[k].T, gas) for k in range(n)])
    assert np.array_equal(mu, z[f"{tag}_mu"])
    lam = np.array([eq.thermal_conductivity(m, gas) for m in mu])
    assert np.array_equal(lam, z[f"{tag}_lam"])
    cons = np.array([eq.prim_to_cons(P[k], gas).as_array() for k in range(n)])
    assert np.array_equal(cons, z[f"{tag}_cons"])


def test_riemann_consistency_and_admissibility(gpu):
    """tests/test_equations.py: f*(U, U, n) = F(U).n for every solver; inadmissible
    states raise AdmissibilityError."""
    from paper_2404_12703_b200 import equations as eq
    gas = eq.GasProperties(gamma=1.4, R=1.0)
    P = eq.PrimitiveState(rho=1.3, vel=(0.2, -0.4, 0.1), p=0.8, T=0.8 / 1.3)
    n = np.array([0.6, 0.0, 0.8])
    F = eq.euler_flux(P, eq.prim_to_cons(P, gas))
    for solver in ("llf", "hllc"):
        assert np.allclose(eq.riemann_flux(P, P, n, gas, solver), F.T @ n, atol=1e-13)
    with pytest.raises(eq.AdmissibilityError):
        eq.riemann_flux(eq.PrimitiveState(rho=-1.0, vel=(0, 0, 0), p=1.0, T=1.0), P, n, gas)
    with pytest.raises(ValueError):
        eq.riemann_flux(P, P, np.array([1.0, 1.0, 0.0]), gas)


def test_mms_source_matches_reference(gpu):
    """testcases.mms_source vs the reference's values (device sin/cos: <= a few ulp)."""
    from paper_2404_12703_b200.testcases import ManufacturedSolution, mms_source
    z = golden("physics_points")
    S = mms_source(z["mms_x"], float(z["mms_t"]), _gas(z["mms_gas"]),
                   ManufacturedSolution(amplitude=0.1, speed=1.0))
    ref = z["mms_S"]
    assert np.max(np.abs(S - ref)) <= 1e-14 * np.max(np.abs(ref))
    one = mms_source(z["mms_x"][0], float(z["mms_t"]), _gas(z["mms_gas"]))
    assert one.shape == (5,)


def test_rk_step_host_arrays_bitwise(gpu):
    """rk_step with the reference's numpy signature: the stage update equals the
    reference's numpy order (src/timedisc.py:132-137) bit for bit, work included."""
    from paper_2404_12703_b200.timedisc import get_scheme, rk_step
    rng = np.random.default_rng(4)
    for name in ("carpenter-kennedy-5-4", "niegemann-14-4"):
        sc = get_scheme(name)
        M = rng.standard_normal((6, 6)) * 0.3
        y = rng.standard_normal(6)
        work = np.zeros(6)
        y_ref, w_ref = y.copy(), np.zeros(6)
        calls = []
        rk_step(y, 0.1, 0.05, lambda u, t: calls.append(t) or M @ u, sc, work)
        for i in range(sc.stages):          # the reference's numpy stage, restated
            Ut = M @ y_ref
            if i == 0:
                w_ref[...] = 0.05 * Ut
            else:
                w_ref *= sc.A[i]
                w_ref += 0.05 * Ut
            y_ref += sc.B[i] * w_ref
        assert np.array_equal(y, y_ref) and np.array_equal(work, w_ref)
        assert np.allclose(calls, [0.1 + c * 0.05 for c in sc.c])
    with pytest.raises(RuntimeError, match="RK stage 0"):
        rk_step(np.ones(2), 0.0, 0.1, lambda u, t: 1 / 0, get_scheme("carpenter-kennedy-5-4"))
    with pytest.raises(ValueError):
        rk_step(np.ones(2), 0.0, -0.1, lambda u, t: u, get_scheme("carpenter-kennedy-5-4"))
