"""The reference's own operator / shock / time-integration tests, run against the
B200 path through the same Python API (reference pkg/tests/test_operator.py,
test_shock.py, test_timedisc.py, test_acceptance.py criteria 2, 3, 8).
Tolerances are the reference's."""

import numpy as np
import pytest

from conftest import make_worker
from paper_2404_12703_b200 import mesh as mm
from paper_2404_12703_b200.basis import LGL, build_basis
from paper_2404_12703_b200.config import RunConfig
from paper_2404_12703_b200.equations import RIEMANN_LLF, GasProperties
from paper_2404_12703_b200.operator import Domain, _orient, k_surf_int
from paper_2404_12703_b200.shock import (ShockConfig, blend, fv_subcell_operator,
                                         indicator_alpha, modal_threshold,
                                         subcell_interface_metrics)
from paper_2404_12703_b200.testcases import TGVSetup, freestream_init, tgv_init

pytestmark = pytest.mark.gpu

UNIT = dict(x0=-1.0, x1=1.0, y0=-1.0, y1=1.0, z0=-1.0, z1=1.0)
BALANCED = dict(rgas=1.0)
GAS = GasProperties(gamma=1.4, R=1.0)


def cfgd(**kw):
    base = dict(testcase="freestream", n=3, meshx=2, meshy=2, meshz=2, tend=1.0,
                analyzeinterval=0, **UNIT, **BALANCED)
    base.update(kw)
    return RunConfig(**base)


def box(cfg):
    m = mm.generate_box_mesh(cfg.meshx, cfg.meshy, cfg.meshz,
                             [(cfg.x0, cfg.x1), (cfg.y0, cfg.y1), (cfg.z0, cfg.z1)],
                             (cfg.periodicx, cfg.periodicy, cfg.periodicz))
    return mm.curve_mesh(m, cfg.curveamplitude) if cfg.curveamplitude else m


# ---- tests/test_operator.py -------------------------------------------------------

@pytest.mark.parametrize("op,nt", [("standard", "GL"), ("standard", "LGL"), ("split", "LGL")])
@pytest.mark.parametrize("mu", [0.0, 0.01])
def test_free_stream_ut_zero(gpu, op, nt, mu):
    cfg = cfgd(nodetype=nt, operator=op, curveamplitude=0.08, muref=mu)
    w = make_worker(cfg, box(cfg))
    assert np.max(np.abs(w.evaluate_rhs(0.0))) < 1e-12


def test_free_stream_with_all_orientation_codes(gpu):
    m = mm.curve_mesh(mm.permute_element_axes(
        mm.generate_box_mesh(3, 3, 3, [(-1.0, 1.0)] * 3, (True,) * 3), 13, "flip_xy"), 0.05)
    cfg = cfgd(meshx=3, meshy=3, meshz=3, operator="split", nodetype="LGL", muref=0.01)
    w = make_worker(cfg, m)
    assert np.max(np.abs(w.evaluate_rhs(0.0))) < 5e-12


def test_linear_wave_volume_divergence_exact(gpu):
    cfg = cfgd(operator="standard", nodetype="GL", periodicx=False)
    w = make_worker(cfg, box(cfg))
    d = w.domain
    x = d.x[..., 0]
    rho = 2.0 + 0.1 * x
    d.U[..., 0] = rho
    d.U[..., 1] = rho
    d.U[..., 2] = 0.0
    d.U[..., 3] = 0.0
    d.U[..., 4] = 1.0 / 0.4 + 0.5 * rho
    for tag, xv in ((1, -1.0), (2, 1.0)):
        r = 2.0 + 0.1 * xv
        d.bc_states[tag] = [r, r, 0.0, 0.0, 2.5 + 0.5 * r]
    Ut = w.evaluate_rhs(0.0)
    assert np.max(np.abs(Ut[..., 0] + 0.1)) < 1e-12
    assert np.max(np.abs(Ut[..., 1] + 0.1)) < 1e-12
    assert np.max(np.abs(Ut[..., 2])) < 1e-12
    assert np.max(np.abs(Ut[..., 4] + 0.05)) < 1e-12


def test_prolong_face_values(gpu):
    cfg = cfgd(n=2, nodetype="GL", operator="standard")
    w = make_worker(cfg, box(cfg))
    d = w.domain
    xi = d.basis.nodes
    d.U[...] = 0.0
    d.U[..., 0] = xi[None, None, None, :] ** 2
    d.prolong(mpi=False)
    for sl in range(d.ns):
        if d.mesh.side_loc_p[d.side_global[sl]] // 2 == 0:
            assert np.max(np.abs(d.UL[sl, :, :, 0] - 1.0)) < 1e-13


def test_prolong_lgl_is_copy(gpu):
    cfg = cfgd(n=3, nodetype="LGL", operator="split")
    w = make_worker(cfg, box(cfg))
    d = w.domain
    d.U[...] = np.random.default_rng(0).standard_normal(d.U.shape)
    d.prolong(mpi=False)
    for sl in range(d.ns):
        sg = d.side_global[sl]
        ep, loc = d.mesh.side_elem_p[sg], d.mesh.side_loc_p[sg]
        if loc == 1:
            assert np.array_equal(d.UL[sl], d.U[ep - d.lo, :, :, -1, :])


def _single_elem_domain(N=1):
    b = build_basis(N, LGL)
    m = mm.generate_box_mesh(1, 1, 1, [(-1.0, 1.0)] * 3, (True,) * 3)
    mm.compute_metrics(m, b)
    return m, b, Domain(m, b, GasProperties())


def test_surf_int_pencil_and_paper(gpu):
    """tests/test_operator.py:100-118: the raw k_surf_int call of the reference."""
    m, b, d = _single_elem_domain(1)
    loc_of_side = {int(m.side_loc_p[d.side_global[s]]): s for s in range(d.ns)}
    fstar = np.zeros_like(d.fstar)
    fstar[loc_of_side[1], :, :, 0] = 1.0
    Ut = np.zeros_like(d.Ut)
    k_surf_int(fstar, d.ef_side, d.ef_sign, d.ef_orient, b.lhat_minus, b.lhat_plus, Ut)
    # the Domain method gives the same field
    d.fstar[...] = fstar
    d.Ut[...] = 0.0
    d.surf_int()
    assert np.array_equal(d.Ut, Ut)
    assert np.allclose(Ut[0, :, :, 0, 0], -1.0)
    assert np.allclose(Ut[0, :, :, 1, 0], 1.0)
    assert np.max(np.abs(Ut[..., 1:])) == 0.0


def test_surf_int_gather_matches_scatter_reference(gpu):
    mesh = mm.permute_element_axes(mm.generate_box_mesh(3, 3, 3, [(-1.0, 1.0)] * 3, (True,) * 3),
                                   13, "flip_xy")
    b = build_basis(3, LGL)
    mm.compute_metrics(mesh, b)
    d = Domain(mesh, b, GasProperties())
    assert {int(mesh.side_orient[s]) for s in range(mesh.n_sides)} == {0, 1, 2, 3}
    fstar = 0.01 * np.random.default_rng(42).standard_normal(d.fstar.shape)
    Ut = np.zeros_like(d.Ut)
    k_surf_int(fstar, d.ef_side, d.ef_sign, d.ef_orient, b.lhat_minus, b.lhat_plus, Ut)
    # independent side-loop scatter (reference tests/helpers.py:36-63)
    ref = np.zeros_like(d.Ut)
    N = b.N
    for sl, sg in enumerate(d.side_global):
        roles = [(mesh.side_elem_p[sg], mesh.side_loc_p[sg], 1.0, 0)]
        if mesh.side_elem_r[sg] >= 0:
            roles.append((mesh.side_elem_r[sg], mesh.side_loc_r[sg], -1.0, mesh.side_orient[sg]))
        for elem, loc, sign, code in roles:
            for p in range(N + 1):
                for q in range(N + 1):
                    line, dd, plus = mm.side_mapping(loc, code, p, q, N)
                    lh = b.lhat_plus if plus else b.lhat_minus
                    for mm_ in range(N + 1):
                        i, j, k = line[mm_]
                        ref[elem, k, j, i] += sign * lh[line[mm_][dd]] * fstar[sl, q, p]
    assert np.max(np.abs(Ut - ref)) <= 1e-15


def test_apply_jac_scales_and_flips(gpu):
    cfg = cfgd()
    w = make_worker(cfg, box(cfg))
    d = w.domain
    d.Ut[...] = 1.0
    d.apply_jac()
    assert np.allclose(d.Ut, -1.0 / d.J[..., None])


def test_lifting_linear_field_exact(gpu):
    cfg = cfgd(operator="standard", nodetype="GL", periodicx=False, muref=0.01)
    w = make_worker(cfg, box(cfg))
    d = w.domain
    x = d.x[..., 0]
    d.U[..., 0] = 1.0
    d.U[..., 1] = x
    d.U[..., 2] = 0.0
    d.U[..., 3] = 0.0
    d.U[..., 4] = 2.5 + 0.5 * x * x
    for tag, xv in ((1, -1.0), (2, 1.0)):
        d.bc_states[tag] = [1.0, xv, 0.0, 0.0, 2.5 + 0.5 * xv * xv]
    w.evaluate_rhs(0.0)
    g = d.g
    assert np.max(np.abs(g[..., 0, 0] - 1.0)) < 1e-12
    assert np.max(np.abs(g[..., 1, 0])) < 1e-12
    assert np.max(np.abs(g[..., 2, 0])) < 1e-12
    assert np.max(np.abs(g[..., :, 1:3])) < 1e-12


def test_lifting_sine_converges(gpu):
    errs = []
    for m in (2, 4, 8):
        cfg = cfgd(meshx=m, meshy=m, meshz=m, operator="split", nodetype="LGL", muref=0.01, n=3)
        w = make_worker(cfg, box(cfg))
        d = w.domain
        x = d.x[..., 0]
        d.U[..., 0] = 1.0
        d.U[..., 1] = np.sin(np.pi * x)
        d.U[..., 2:4] = 0.0
        d.U[..., 4] = 2.5 + 0.5 * np.sin(np.pi * x) ** 2
        w.evaluate_rhs(0.0)
        e = d.g[..., 0, 0] - np.pi * np.cos(np.pi * x)
        errs.append(np.sqrt(np.mean(e ** 2)))
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert rates[-1] >= 2.9, (errs, rates)


def test_constant_field_gradients_vanish(gpu):
    cfg = cfgd(curveamplitude=0.08, muref=0.01, operator="split", nodetype="LGL")
    w = make_worker(cfg, box(cfg))
    w.evaluate_rhs(0.0)
    assert np.max(np.abs(w.domain.g)) < 1e-13


def test_compute_dt_uniform_mesh_closed_form(gpu):
    cfg = cfgd(n=3, operator="standard", nodetype="GL", x0=0.0, x1=2.0, y0=0.0, y1=2.0,
               z0=0.0, z1=2.0)
    w = make_worker(cfg, box(cfg))
    d = w.domain
    d.U[..., 0] = 1.0
    d.U[..., 1:4] = 0.0
    d.U[..., 4] = 1.0 / 0.4
    d.cons_to_prim()
    expect = 0.9 * 1.0 / (3.0 * 7.0 * np.sqrt(1.4))
    assert abs(d.local_dt(0.9, 0.4) - expect) < 1e-13 * expect


def test_compute_dt_halves_under_refinement(gpu):
    vals = []
    for m in (2, 4):
        cfg = cfgd(meshx=m, meshy=m, meshz=m)
        w = make_worker(cfg, box(cfg))
        w.domain.U[...] = freestream_init(w.domain.x, cfg.gas())
        vals.append(w.domain.local_dt(0.9, 0.4))
    assert abs(vals[0] / vals[1] - 2.0) < 1e-12


def test_inadmissible_state_raises(gpu):
    from paper_2404_12703_b200.equations import AdmissibilityError
    cfg = cfgd()
    w = make_worker(cfg, box(cfg))
    w.domain.U[0, 0, 0, 0, 0] = -1.0
    with pytest.raises(AdmissibilityError):
        w.evaluate_rhs(0.0)


# ---- tests/test_shock.py -----------------------------------------------------------

def lgl_domain(mesh_n=2, N=3, curved=0.0, periodic=(True, True, True), extents=None):
    b = build_basis(N, LGL)
    m = mm.generate_box_mesh(mesh_n, mesh_n, mesh_n, extents or [(-1.0, 1.0)] * 3, periodic)
    if curved:
        m = mm.curve_mesh(m, curved)
    mm.compute_metrics(m, b)
    return Domain(m, b, GAS)


def constant_state(d, rho=1.0, p=1.0):
    d.U[..., 0] = rho
    d.U[..., 1:4] = 0.0
    d.U[..., 4] = p / (GAS.gamma - 1.0)


def test_indicator_constant_element_is_zero(gpu):
    d = lgl_domain()
    constant_state(d)
    assert indicator_alpha(d.U[0], d.basis, ShockConfig(enabled=True)) == 0.0


def test_indicator_high_mode_clamps_to_alpha_max(gpu):
    from paper_2404_12703_b200.basis import legendre
    d = lgl_domain(N=5)
    b = d.basis
    pn, _ = legendre(b.N, b.nodes)
    U = np.zeros((6, 6, 6, 5))
    U[..., 0] = 2.0 + pn[None, None, :] * np.ones((6, 6, 6))
    U[..., 4] = 1.0 / (GAS.gamma - 1.0)
    assert indicator_alpha(U, b, ShockConfig(enabled=True, alpha_max=0.5)) == 0.5


def test_indicator_zero_on_resolved_tgv_field(gpu):
    setup = TGVSetup(mach=0.1, reynolds=1600.0, version=2)
    gas = GasProperties(gamma=1.4, R=287.058)
    b = build_basis(7, LGL)
    mesh = mm.generate_box_mesh(8, 8, 8, setup.domain, (True,) * 3)
    mm.compute_metrics(mesh, b)
    U = tgv_init(setup, mesh.x, gas)
    alphas = np.array([indicator_alpha(U[e], b, ShockConfig(enabled=True), gas.gamma)
                       for e in range(0, mesh.nelem, 7)])
    assert np.mean(alphas == 0.0) >= 0.99


def test_threshold_decreases_with_degree():
    ts = [modal_threshold(N) for N in range(1, 10)]
    assert all(t1 > t2 for t1, t2 in zip(ts, ts[1:]))


@pytest.mark.parametrize("curved", [0.0, 0.1])
def test_fv_residual_zero_for_constant_state(gpu, curved):
    d = lgl_domain(curved=curved)
    constant_state(d)
    d.cons_to_prim()
    d.prolong(mpi=False)
    d.prolong(mpi=True)
    d.fill_flux(d.sides_inner, RIEMANN_LLF)
    fvm = subcell_interface_metrics(d)
    for e in range(d.ne):
        assert np.max(np.abs(fv_subcell_operator(d, e, fvm=fvm))) < 1e-13


def test_fv_conservation_telescopes_to_outer_flux(gpu):
    d = lgl_domain(curved=0.05)
    rng = np.random.default_rng(1)
    constant_state(d)
    d.U[..., 0] += 0.2 * rng.random(d.U.shape[:-1])
    d.U[..., 4] += 0.3 * rng.random(d.U.shape[:-1])
    d.cons_to_prim()
    d.prolong(mpi=False)
    d.fill_flux(d.sides_inner, RIEMANN_LLF)
    fvm = subcell_interface_metrics(d)
    w = d.basis.weights
    wvol = w[None, None, :] * w[None, :, None] * w[:, None, None]
    N = d.N
    for e in range(d.ne):
        R = fv_subcell_operator(d, e, fvm=fvm)
        total = np.einsum("kji,kjiv->v", wvol, R * d.J[e][..., None])
        net = np.zeros(5)
        for loc in range(6):
            s, sign, code = d.ef_side[e, loc], d.ef_sign[e, loc], d.ef_orient[e, loc]
            for a in range(N + 1):
                for bq in range(N + 1):
                    p, q = _orient(code, a, bq, N)
                    net += sign * w[a] * w[bq] * d.fstar[s, q, p]
        assert np.max(np.abs(total + net)) < 1e-12 * max(1.0, np.max(np.abs(net)))


def test_blend_endpoints_and_mean():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((4, 4, 4, 5))
    b = rng.standard_normal((4, 4, 4, 5))
    assert np.array_equal(blend(a, b, 0.0), a)
    assert np.array_equal(blend(a, b, 1.0), b)
    with pytest.raises(ValueError):
        blend(a, b, 1.5)


# ---- tests/test_timedisc.py (device rk_step) ----------------------------------------

@pytest.mark.parametrize("name", ["carpenter-kennedy-5-4", "niegemann-14-4"])
def test_rk_order(gpu, name):
    import torch
    from paper_2404_12703_b200.timedisc import get_scheme, rk_step
    sc = get_scheme(name)
    lam = -1.0 + 0.5j

    def solve(nsteps):
        U = torch.tensor([1.0, 0.0], dtype=torch.float64, device="cuda")
        work = torch.zeros_like(U)
        A = torch.tensor([[lam.real, -lam.imag], [lam.imag, lam.real]], dtype=torch.float64,
                         device="cuda")
        calls = []

        def rhs(u, t):
            calls.append(t)
            return (A @ u).contiguous()
        dt = 1.0 / nsteps
        for n in range(nsteps):
            rk_step(U, n * dt, dt, rhs, sc, work)
        assert len(calls) == nsteps * sc.stages
        return U.cpu().numpy()
    exact = np.exp(lam)
    errs = [abs(complex(*solve(n)) - exact) for n in (10, 20)]
    assert np.log2(errs[0] / errs[1]) >= 3.8


# ---- acceptance criteria 2 and 3 (tests/test_acceptance.py:63-96) ----------------------

def test_criterion_2_free_stream_preservation(gpu):
    from paper_2404_12703_b200.parallel import run_distributed
    ref = freestream_init(np.zeros((1, 3)), RunConfig().gas())[0]
    worst = 0.0
    for op, nt in (("standard", "GL"), ("split", "LGL")):
        for mu in (0.0, 1e-3):
            cfg = RunConfig(testcase="freestream", n=4, nodetype=nt, operator=op, meshx=4,
                            meshy=4, meshz=4, **UNIT, curveamplitude=0.1, muref=mu, tend=1e9,
                            maxsteps=20, analyzeinterval=0)
            res = run_distributed(cfg)
            worst = max(worst, float(np.max(np.abs(res.U - ref))))
    assert worst <= 1e-11, worst


@pytest.mark.parametrize("cap", [False, True])
def test_criterion_3_conservation(gpu, cap):
    from paper_2404_12703_b200.parallel import run_distributed
    two_pi = 2 * np.pi
    cfg = RunConfig(testcase="tgv", n=5, meshx=4, meshy=4, meshz=4, x0=0.0, x1=two_pi, y0=0.0,
                    y1=two_pi, z0=0.0, z1=two_pi, mach=0.1, muref=0.0, maxsteps=100, tend=1e9,
                    analyzeinterval=0, shockcapture=cap, indicator="constant",
                    alphaconst=0.3 if cap else 0.0)
    b = build_basis(5, LGL)
    m = mm.generate_box_mesh(4, 4, 4, [(0.0, two_pi)] * 3, (True,) * 3)
    mm.compute_metrics(m, b)
    wq = b.weights
    dv = m.J * wq[None, None, None, :] * wq[None, None, :, None] * wq[None, :, None, None]
    U0 = tgv_init(TGVSetup(mach=0.1, reynolds=1600.0), m.x, cfg.gas())
    tot0 = np.einsum("ekji,ekjiv->v", dv, U0)
    res = run_distributed(cfg, mesh=m)
    tot1 = np.einsum("ekji,ekjiv->v", dv, res.U)
    scale = max(abs(tot0[0]), abs(tot0[4]))
    assert np.max(np.abs(tot1 - tot0)) / scale <= 1e-11
