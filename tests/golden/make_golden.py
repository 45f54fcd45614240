"""Generate the golden vectors by running the REFERENCE package itself.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz (committed). Nothing on the GPU box reads
/root/reference; the tests read only these fixtures.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from hexdg import testcases  # noqa: E402
from hexdg.basis import build_basis  # noqa: E402
from hexdg.config import RunConfig  # noqa: E402
from hexdg.mesh import (compute_metrics, curve_mesh, generate_box_mesh,  # noqa: E402
                        partition_sfc, permute_element_axes)
from hexdg.operator import Domain  # noqa: E402
from hexdg.parallel import RankWorker, SlotLimiter, Transport  # noqa: E402
from hexdg.shock import subcell_interface_metrics  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TABLE_KEYS = ("side_elem_p", "side_loc_p", "side_elem_r", "side_loc_r", "side_orient",
              "side_bc", "elem_sides", "elem_primary", "grid_index")
DOMAIN_KEYS = ("side_global", "ef_side", "ef_sign", "ef_orient", "rows_inner", "rows_mpi",
               "sides_inner", "sides_mpi_primary", "sides_mpi_replica", "sides_bc", "side_bc")


def save(name, **arrs):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrs)
    print("wrote", name, sum(np.asarray(v).nbytes for v in arrs.values()) // 1024, "KiB raw")


def mesh_spec(**kw):
    return {f"spec_{k}": np.asarray(v) for k, v in kw.items()}


def build_mesh(nx, ny, nz, extents, periodic, flips=(), curve=0.0):
    m = generate_box_mesh(nx, ny, nz, extents, periodic)
    for e, k in flips:
        m = permute_element_axes(m, e, k)
    if curve:
        m = curve_mesh(m, curve)
    return m


def basis_golden():
    out = {}
    for N in range(1, 9):
        for nt in ("GL", "LGL"):
            b = build_basis(N, nt)
            for f in ("nodes", "weights", "D", "Dhat", "Dsplit", "l_minus", "l_plus",
                      "lhat_minus", "lhat_plus", "vandermonde_modal", "geom_to_solution"):
                out[f"{nt}{N}_{f}"] = getattr(b, f)
    save("basis", **out)


def tables_golden():
    rng = np.random.default_rng(7)
    cases = {
        "orient3": dict(n=(3, 3, 3), ext=[(-1.0, 1.0)] * 3, per=(True,) * 3,
                        flips=[(13, "flip_xy")]),
        "walls432": dict(n=(4, 3, 2), ext=[(0.0, 1.0), (-1.0, 2.0), (0.0, 3.0)],
                         per=(False, True, False), flips=[]),
        "randflip4": dict(n=(4, 4, 4), ext=[(0.0, 1.0)] * 3, per=(True, True, False),
                          flips=[(int(rng.integers(64)), ("flip_xy", "flip_xz", "flip_yz")[rng.integers(3)])
                                 for _ in range(40)]),
    }
    for name, c in cases.items():
        m = build_mesh(*c["n"], c["ext"], c["per"], c["flips"])
        out = {k: getattr(m, k) for k in TABLE_KEYS}
        out["flip_elems"] = np.array([e for e, _ in c["flips"]], dtype=np.int64)
        out["flip_kinds"] = np.array([k for _, k in c["flips"]])
        out.update(mesh_spec(n=c["n"], ext=c["ext"], per=c["per"]))
        b = build_basis(3, "LGL")
        mc = curve_mesh(m, 0.05)
        compute_metrics(mc, b)
        out.update(J=mc.J, Ja=mc.Ja, x=mc.x, face_normal=mc.face_normal, face_s=mc.face_s)
        nr = 3
        parts = partition_sfc(mc, nr)
        elem_rank = np.empty(mc.nelem, dtype=np.int64)
        for p in parts:
            elem_rank[p.lo:p.hi] = p.rank
            out[f"part{p.rank}_lo"] = np.int64(p.lo)
            out[f"part{p.rank}_hi"] = np.int64(p.hi)
            for k, v in p.neighbors.items():
                out[f"part{p.rank}_nbr{k}"] = v
        for r in range(nr):
            d = Domain(mc, b, testcases.GasProperties() if hasattr(testcases, "GasProperties")
                       else __import__("hexdg.equations", fromlist=["x"]).GasProperties(),
                       parts[r].lo, parts[r].hi, elem_rank, r)
            for k in DOMAIN_KEYS:
                out[f"dom{r}_{k}"] = np.asarray(getattr(d, k))
            for nb, info in d.neighbors.items():
                out[f"dom{r}_nbr{nb}_sides"] = info["sides"]
                out[f"dom{r}_nbr{nb}_is_primary"] = info["is_primary"]
        save("tables_" + name, **out)


def random_state(shape, rng, mach=0.3):
    rho = 1.0 + 0.2 * rng.random(shape)
    u = mach * rng.standard_normal(shape + (3,))
    p = 1.0 + 0.2 * rng.random(shape)
    U = np.empty(shape + (5,))
    U[..., 0] = rho
    U[..., 1:4] = rho[..., None] * u
    U[..., 4] = p / 0.4 + 0.5 * rho * np.sum(u * u, axis=-1)
    return U


def make_worker(cfg, mesh):
    basis = build_basis(cfg.n, cfg.nodetype)
    compute_metrics(mesh, basis)
    parts = partition_sfc(mesh, 1)
    return RankWorker(0, mesh, basis, cfg.gas(), parts[0], np.zeros(mesh.nelem, dtype=np.int64),
                      cfg, Transport(1), SlotLimiter(1), testcases.build_case(cfg))


def dump_domain(w):
    d = w.domain
    out = {k: np.asarray(getattr(d, k)) for k in DOMAIN_KEYS}
    out.update(Ja=d.Ja, J=d.J, x=d.x, nvec=d.nvec, ssurf=d.ssurf, bc_states=d.bc_states)
    return out


def rhs_case(name, cfg, mesh, U=None, seed=0, t=0.0, bc=None, steps=0, mesh_desc=None,
             lean=False):
    w = make_worker(cfg, mesh)
    d = w.domain
    if U is not None:
        d.U[...] = U(d.x) if callable(U) else U
    if bc is not None:
        d.bc_states[...] = bc
    out = dump_domain(w)
    out["U0"] = d.U.copy()
    Ut = w.evaluate_rhs(t).copy()
    out.update(Ut=Ut, fstar=d.fstar.copy(), alpha=w.alpha.copy(), t=np.float64(t))
    if not lean:   # lean: Ut / fstar / trajectory only (the intermediates are in the other cases)
        out.update(prim=d.prim.copy(), UL=d.UL.copy(), UR=d.UR.copy())
    if d.viscous and not lean:
        out.update(g=d.g.copy(), gL=d.gL.copy(), gR=d.gR.copy(), vstar=d.vstar.copy(),
                   Fvis=d.Fvis.copy())
    if cfg.shockcapture:
        f0, f1, f2 = subcell_interface_metrics(d)
        out.update(fvm0=f0, fvm1=f1, fvm2=f2)
    out["dt"] = np.float64(d.local_dt(cfg.cfl, cfg.cflvisc))
    for f in ("n", "nodetype", "operator", "riemann", "rkscheme", "cfl", "cflvisc", "shockcapture",
              "alphamax", "alphamin", "indicator", "alphaconst", "gamma", "rgas", "prandtl",
              "muref", "tref", "viscosity", "testcase", "mmsamplitude", "mmsspeed"):
        out["cfg_" + f] = np.asarray(getattr(cfg, f))
    out.update(mesh_desc or {})
    if steps:
        # reference time loop (RankWorker.run without analysis)
        from hexdg.timedisc import rk_step
        d.U[...] = out["U0"]
        dts = []
        tt = 0.0
        for _ in range(steps):
            dt = w._compute_dt()
            rk_step(d.U, tt, dt, lambda U, ts: w.evaluate_rhs(ts), w.scheme, w.rk_work)
            tt += dt
            dts.append(dt)
        out.update(U_final=d.U.copy(), dts=np.array(dts), t_final=np.float64(tt))
    save("rhs_" + name, **out)


def orient_mesh(curve=0.05):
    m = generate_box_mesh(3, 3, 3, [(-1.0, 1.0)] * 3, (True,) * 3)
    m = permute_element_axes(m, 13, "flip_xy")
    return curve_mesh(m, curve)


def desc(n, ext, per, flips=(), curve=0.0):
    return {"mesh_n": np.array(n), "mesh_ext": np.array(ext, dtype=float),
            "mesh_per": np.array(per), "mesh_flip_e": np.array([e for e, _ in flips], dtype=np.int64),
            "mesh_flip_k": np.array([k for _, k in flips] or [""]), "mesh_curve": np.float64(curve)}


def rhs_golden():
    rng = np.random.default_rng(11)
    U3 = random_state((27, 4, 4, 4), rng)
    UNIT = dict(x0=-1.0, x1=1.0, y0=-1.0, y1=1.0, z0=-1.0, z1=1.0)
    od = desc((3, 3, 3), [(-1.0, 1.0)] * 3, (True,) * 3, [(13, "flip_xy")], 0.05)
    # A: Euler, split, LGL N=3, all orientation codes, curved
    rhs_case("euler_split_n3", RunConfig(testcase="freestream", n=3, rgas=1.0, **UNIT),
             orient_mesh(), U3, mesh_desc=od)
    # B: NS (constant mu), split, same mesh
    rhs_case("ns_split_n3", RunConfig(testcase="freestream", n=3, rgas=1.0, muref=0.01, **UNIT),
             orient_mesh(), U3, mesh_desc=od)
    # C: NS Sutherland, standard form on GL nodes, non-periodic x walls (Dirichlet BC)
    m = curve_mesh(generate_box_mesh(2, 2, 2, [(-1.0, 1.0)] * 3, (False, True, True)), 0.05)
    U = random_state((8, 4, 4, 4), rng)
    bc = np.zeros((8, 5))
    bc[1] = random_state((1,), rng)[0]
    bc[2] = random_state((1,), rng)[0]
    rhs_case("ns_std_gl_walls_n3",
             RunConfig(testcase="freestream", n=3, nodetype="GL", operator="standard", rgas=1.0,
                       muref=0.02, viscosity="sutherland", tref=2.0, periodicx=False, **UNIT),
             m, U, bc=bc, mesh_desc=desc((2, 2, 2), [(-1.0, 1.0)] * 3, (False, True, True), (), 0.05))
    # D: Euler, standard form, LGL N=4, HLLC, all orientations
    U4 = random_state((27, 5, 5, 5), rng)
    rhs_case("euler_std_hllc_n4",
             RunConfig(testcase="freestream", n=4, operator="standard", riemann="hllc", rgas=1.0,
                       **UNIT), orient_mesh(), U4, mesh_desc=od)
    # E: TGV Ma 1.25 NS Sutherland N=5 with FV everywhere (alpha const 0.3), curved
    gas_t0 = 1.0 / (1.4 * 1.25 ** 2 * 287.058)
    two_pi = 2 * np.pi
    tgv_ext = dict(x0=0.0, x1=two_pi, y0=0.0, y1=two_pi, z0=0.0, z1=two_pi)
    m = curve_mesh(generate_box_mesh(2, 2, 2, [(0.0, two_pi)] * 3, (True,) * 3), 0.05)
    rhs_case("tgv_fv_const_n5",
             RunConfig(testcase="tgv", n=5, mach=1.25, muref=1.0 / 1600.0, viscosity="sutherland",
                       tref=gas_t0, shockcapture=True, indicator="constant", alphaconst=0.3,
                       **tgv_ext), m,
             mesh_desc=desc((2, 2, 2), [(0.0, two_pi)] * 3, (True,) * 3, (), 0.05))
    # F: Euler split N=5, Hennemann indicator with a discontinuous state (some alpha > 0), HLLC FV
    m = curve_mesh(generate_box_mesh(2, 2, 2, [(-1.0, 1.0)] * 3, (True,) * 3), 0.05)

    def sodish(x):
        rho = np.where(x[..., 0] < 0.13, 1.0, 0.125) + 0.05 * np.sin(3 * x[..., 1])
        p = np.where(x[..., 0] < 0.13, 1.0, 0.1)
        U = np.zeros(x.shape[:-1] + (5,))
        U[..., 0] = rho
        U[..., 1] = 0.1 * rho
        U[..., 4] = p / 0.4 + 0.5 * rho * 0.01
        return U
    rhs_case("euler_hennemann_n5",
             RunConfig(testcase="freestream", n=5, riemann="hllc", shockcapture=True, rgas=1.0,
                       alphamax=0.6, **UNIT), m, sodish,
             mesh_desc=desc((2, 2, 2), [(-1.0, 1.0)] * 3, (True,) * 3, (), 0.05))
    # G: C2 miniature: TGV Ma 0.1 NS split N=7, 2^3
    m = generate_box_mesh(2, 2, 2, [(0.0, two_pi)] * 3, (True,) * 3)
    rhs_case("tgv_ns_split_n7",
             RunConfig(testcase="tgv", n=7, mach=0.1, muref=1.0 / 1600.0, **tgv_ext), m,
             mesh_desc=desc((2, 2, 2), [(0.0, two_pi)] * 3, (True,) * 3))
    # H: C1 miniature: MMS Euler, GL standard N=3, 4^3 on [-1,1]^3, source at t = 0.3
    m = generate_box_mesh(4, 4, 4, [(-1.0, 1.0)] * 3, (True,) * 3)
    rhs_case("mms_gl_std_n3",
             RunConfig(testcase="mms", n=3, nodetype="GL", operator="standard",
                       rkscheme="carpenter-kennedy-5-4", **UNIT), m, t=0.3,
             mesh_desc=desc((4, 4, 4), [(-1.0, 1.0)] * 3, (True,) * 3))
    # I: 100-step trajectory: TGV NS split N=3 3^3, curved all-orientation mesh, niegemann-14
    m = generate_box_mesh(3, 3, 3, [(0.0, two_pi)] * 3, (True,) * 3)
    m = curve_mesh(permute_element_axes(m, 13, "flip_xz"), 0.05)
    rhs_case("traj_tgv_ns_n3",
             RunConfig(testcase="tgv", n=3, mach=0.1, muref=1.0 / 1600.0, **tgv_ext), m, steps=100,
             mesh_desc=desc((3, 3, 3), [(0.0, two_pi)] * 3, (True,) * 3, [(13, "flip_xz")], 0.05))
    # J: 20-step trajectory with FV blending (alpha 0.3) and 14-stage RK
    m = generate_box_mesh(2, 2, 2, [(0.0, two_pi)] * 3, (True,) * 3)
    rhs_case("traj_tgv_fv_n4",
             RunConfig(testcase="tgv", n=4, mach=1.25, muref=0.0, shockcapture=True,
                       indicator="constant", alphaconst=0.3, rkscheme="niegemann-14-4", **tgv_ext),
             m, steps=20, mesh_desc=desc((2, 2, 2), [(0.0, two_pi)] * 3, (True,) * 3))


def c4_golden():
    """The benchmark configurations in miniature, produced by the reference:

    * C4: N=4 NS split (TGV Ma 0.1), every element flipped with p=0.5 (kind
      uniform, default_rng(0), sequential permute_element_axes), curve 0.05, 4^3,
      with a perturbed velocity field; one RHS + a 20-step trajectory.
    * C2: TGV Ma 0.1 NS split N=7 on a curved 3^3 mesh, a random double-axis
      flip drawn 12 times (elements sampled with replacement), perturbed velocity;
      a 100-step trajectory (the dt sequence is stored so the GPU can replay it).
    """
    two_pi = 2 * np.pi
    tgv_ext = dict(x0=0.0, x1=two_pi, y0=0.0, y1=two_pi, z0=0.0, z1=two_pi)
    rng = np.random.default_rng(0)
    ne = 4 ** 3
    pick = rng.random(ne) < 0.5
    kind_ix = rng.integers(0, 3, ne)
    names = ("flip_xy", "flip_xz", "flip_yz")
    flips = [(int(e), names[kind_ix[e]]) for e in np.flatnonzero(pick)]
    m = build_mesh(4, 4, 4, [(0.0, two_pi)] * 3, (True,) * 3, flips, 0.05)
    prng = np.random.default_rng(3)

    def perturbed(cfg):
        def f(x):
            from hexdg.testcases import build_case
            U = build_case(cfg)[0](x, cfg.gas())
            U[..., 1:4] += 0.05 * prng.standard_normal(U[..., 1:4].shape)
            return U
        return f
    cfg = RunConfig(testcase="tgv", n=4, mach=0.1, muref=1.0 / 1600.0, **tgv_ext)
    rhs_case("c4_ns_split_n4", cfg, m, perturbed(cfg), steps=20, lean=True,
             mesh_desc=desc((4, 4, 4), [(0.0, two_pi)] * 3, (True,) * 3, flips, 0.05))
    rng = np.random.default_rng(9)
    flips7 = [(int(rng.integers(27)), names[rng.integers(3)]) for _ in range(12)]
    m7 = build_mesh(3, 3, 3, [(0.0, two_pi)] * 3, (True,) * 3, flips7, 0.03)
    cfg7 = RunConfig(testcase="tgv", n=7, mach=0.1, muref=1.0 / 1600.0, **tgv_ext)
    rhs_case("traj_c2_ns_n7", cfg7, m7, perturbed(cfg7), steps=100, lean=True,
             mesh_desc=desc((3, 3, 3), [(0.0, two_pi)] * 3, (True,) * 3, flips7, 0.03))


def physics_golden():
    """The array-level physics API (src/equations.py:288-383) and the MMS source
    (src/testcases.py:73-82) on random admissible states, by the reference."""
    from hexdg import equations as eq
    rng = np.random.default_rng(31)
    out = {}
    gases = {"const": eq.GasProperties(gamma=1.4, R=1.0, mu_ref=0.01),
             "suth": eq.GasProperties(gamma=1.4, R=287.058, mu_ref=1e-3, T_ref=1.2,
                                      viscosity_law=eq.SUTHERLAND)}
    n = 16
    for tag, gas in gases.items():
        prims = []
        for _ in range(2 * n):
            rho = float(rng.uniform(0.1, 5.0))
            vel = tuple(float(v) for v in rng.uniform(-2.0, 2.0, 3))
            p = float(rng.uniform(0.1, 5.0))
            prims.append(eq.PrimitiveState(rho=rho, vel=vel, p=p, T=p / (rho * gas.R)))
        normals = rng.standard_normal((n, 3))
        normals /= np.linalg.norm(normals, axis=1)[:, None]
        grads = rng.standard_normal((n, 3, eq.N_LIFT))
        metrics = rng.standard_normal((n, 3))
        out[f"{tag}_prims"] = np.array([[P.rho, *P.vel, P.p, P.T] for P in prims])
        out[f"{tag}_normals"], out[f"{tag}_grads"], out[f"{tag}_metrics"] = normals, grads, metrics
        for solver in ("llf", "hllc"):
            out[f"{tag}_riemann_{solver}"] = np.array(
                [eq.riemann_flux(prims[2 * k], prims[2 * k + 1], normals[k], gas, solver)
                 for k in range(n)])
        out[f"{tag}_kep"] = np.array([eq.split_flux_twopoint(prims[2 * k], prims[2 * k + 1],
                                                             metrics[k], gas) for k in range(n)])
        out[f"{tag}_euler"] = np.array([eq.euler_flux(prims[k], eq.prim_to_cons(prims[k], gas))
                                        for k in range(n)])
        out[f"{tag}_viscous"] = np.array([eq.viscous_flux(prims[k], grads[k], gas)
                                          for k in range(n)])
        out[f"{tag}_mu"] = np.array([eq.viscosity(prims[k].T, gas) for k in range(n)])
        out[f"{tag}_lam"] = np.array([eq.thermal_conductivity(out[f"{tag}_mu"][k], gas)
                                      for k in range(n)])
        out[f"{tag}_cons"] = np.array([eq.prim_to_cons(prims[k], gas).as_array()
                                       for k in range(n)])
        out[f"{tag}_gas"] = np.array([gas.gamma, gas.R, gas.Pr, gas.mu_ref, gas.T_ref,
                                      gas.viscosity_law])
    gas = eq.GasProperties(gamma=1.4, R=287.058, mu_ref=0.002)
    mms = testcases.ManufacturedSolution(amplitude=0.1, speed=1.0)
    x = rng.uniform(-1.0, 1.0, (64, 3))
    out["mms_x"], out["mms_t"] = x, np.float64(0.37)
    out["mms_S"] = testcases.mms_source(x, 0.37, gas, mms)
    out["mms_gas"] = np.array([gas.gamma, gas.R, gas.Pr, gas.mu_ref, gas.T_ref, 0.0])
    save("physics_points", **out)


def analysis_golden():
    """k_analysis_partials rows on lifted states + a whole run_distributed time
    loop with analysis every 2 steps (series rows, final U) + the reference's
    own HDGF snapshot / series CSV bytes."""
    from hexdg import io as hio
    from hexdg.parallel import run_distributed
    two_pi = 2 * np.pi
    tgv_ext = dict(x0=0.0, x1=two_pi, y0=0.0, y1=two_pi, z0=0.0, z1=two_pi)
    rng = np.random.default_rng(21)
    out = {}
    # viscous TGV N=4 2^3 curved with a perturbed state (lifted gradients from evaluate_rhs)
    cfg = RunConfig(testcase="tgv", n=4, mach=0.3, muref=1.0 / 1600.0, **tgv_ext)
    m = curve_mesh(generate_box_mesh(2, 2, 2, [(0.0, two_pi)] * 3, (True,) * 3), 0.05)
    w = make_worker(cfg, m)
    d = w.domain
    d.U[..., 1:4] += 0.05 * rng.standard_normal(d.U[..., 1:4].shape)
    w.evaluate_rhs(0.0)
    setup = w.case_setup
    out.update(ns_U=d.U.copy(), ns_g=d.g.copy(), ns_mu0=np.float64(setup.mu0()),
               ns_partials=testcases.analysis_partials(d, setup.mu0()))
    q = testcases.reduce_tgv_quantities(out["ns_partials"], setup)
    out.update({"ns_q_" + k: np.float64(v) for k, v in q.items()})
    # Euler (no gradients), mu0 -> 1.0 inside analysis_partials
    cfg = RunConfig(testcase="tgv", n=3, mach=0.3, **tgv_ext)
    w = make_worker(cfg, generate_box_mesh(2, 2, 2, [(0.0, two_pi)] * 3, (True,) * 3))
    w.domain.U[..., 0] += 0.1 * rng.random(w.domain.U[..., 0].shape)
    out.update(eu_U=w.domain.U.copy(), eu_partials=testcases.analysis_partials(w.domain, 0.0))
    save("analysis_partials", **out)
    # the reference time loop with analysis (RankWorker.run, src/parallel.py:606-665)
    series = {}
    for visc in (True, False):
        cfg = RunConfig(testcase="tgv", n=3, mach=0.1, muref=(1.0 / 1600.0) if visc else 0.0,
                        meshx=3, meshy=3, meshz=3, maxsteps=5, analyzeinterval=2, tend=1e9,
                        **tgv_ext)
        res = run_distributed(cfg)
        tag = "ns" if visc else "eu"
        cols = hio.SERIES_COLUMNS + ["volume"]
        series[tag + "_series"] = np.array([[row.get(c, 0.0) for c in cols] for row in res.series])
        series[tag + "_U"] = res.U
        series[tag + "_t"] = np.float64(res.t)
        series["columns"] = np.array(cols)
        path = os.path.join(OUT, f"series_{tag}.csv")
        hio.write_series_csv(path, res.series)
        print("wrote", path)
    save("run_series", **series)
    # HDGF snapshot bytes written by the reference (N=1, 3 elements, alpha given)
    U = rng.standard_normal((3, 2, 2, 2, 5))
    hio.write_snapshot(os.path.join(OUT, "snapshot_ref.hdgf"), U, 0.125, alpha=np.array([0.0, 0.3, 1.0]))
    np.save(os.path.join(OUT, "snapshot_ref_U.npy"), U)


if __name__ == "__main__":
    parts = sys.argv[1:] or ["basis", "tables", "rhs", "analysis", "c4", "physics"]
    if "basis" in parts:
        basis_golden()
    if "tables" in parts:
        tables_golden()
    if "rhs" in parts:
        rhs_golden()
    if "analysis" in parts:
        analysis_golden()
    if "c4" in parts:
        c4_golden()
    if "physics" in parts:
        physics_golden()
