"""Drop-in surface: every name of the reference's hot-path Python API
exists here with a compatible signature (the reference's parameters, in order, as a
prefix; extra parameters only with defaults). CPU only; the comparison against the
reference runs when its source tree is present (this build container)."""

import importlib
import inspect
import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"

NAMES = {
    "basis": ["build_basis", "Basis1D"],
    "mesh": ["generate_box_mesh", "curve_mesh", "permute_element_axes", "compute_metrics",
             "partition_sfc", "write_mesh_cache", "load_mesh_cache", "Mesh", "Partition",
             "MeshError"],
    "equations": ["GasProperties", "AdmissibilityError", "ConservedState", "PrimitiveState",
                  "cons_to_prim", "prim_to_cons", "viscosity", "thermal_conductivity",
                  "euler_flux", "viscous_flux", "riemann_flux", "split_flux_twopoint",
                  "br1_lifting_flux", "CONST_VISCOSITY", "SUTHERLAND", "N_LIFT"],
    "operator": ["Domain", "k_surf_int", "OperatorError"],
    "parallel": ["RankWorker", "Transport", "SlotLimiter", "run_distributed", "Scheduler",
                 "TraceRow", "ProtocolError", "NumericalFailure", "RunResult", "PRIO_LOW",
                 "PRIO_MID", "PRIO_TOP", "PHASE_TRACES", "PHASE_FLUXES"],
    "timedisc": ["rk_step", "get_scheme", "SCHEMES", "RKScheme"],
    "shock": ["ShockConfig", "indicator_alpha", "subcell_interface_metrics",
              "fv_subcell_operator", "blend", "modal_threshold"],
    "testcases": ["mms_source", "tgv_init", "sod_init", "freestream_init", "TGVSetup",
                  "ManufacturedSolution", "analysis_partials", "reduce_tgv_quantities",
                  "analyze_tgv", "build_case", "run_convergence_study", "l2_error_density"],
    "io": ["write_snapshot", "read_snapshot", "write_series_csv"],
    "config": ["RunConfig", "ConfigError"],
}
DOMAIN_METHODS = ["cons_to_prim", "prolong", "apply_bc_traces", "fill_flux", "lift_fill",
                  "lift_volume", "lift_finish", "lift_gradients", "prolong_grad", "vol_int",
                  "surf_int", "apply_jac", "local_dt"]
WORKER_METHODS = ["evaluate_rhs", "run", "analyze"]
SCHEDULER_METHODS = ["add", "run"]
TRANSPORT_METHODS = ["send", "poll", "wait", "wait_any", "has_message", "abort"]


def _compatible(ref, ours):
    try:
        sr, so = inspect.signature(ref), inspect.signature(ours)
    except (TypeError, ValueError):
        return True
    rp, op = list(sr.parameters.values()), list(so.parameters.values())
    if [p.name for p in op[:len(rp)]] != [p.name for p in rp]:
        return False
    return all(p.default is not inspect.Parameter.empty or p.kind in
               (p.VAR_POSITIONAL, p.VAR_KEYWORD) for p in op[len(rp):])


@pytest.mark.parametrize("mod", sorted(NAMES))
def test_names_exist(mod):
    m = importlib.import_module("paper_2404_12703_b200." + mod)
    missing = [n for n in NAMES[mod] if not hasattr(m, n)]
    assert not missing, missing


def test_methods_exist():
    from paper_2404_12703_b200 import operator, parallel
    for cls, names in ((operator.Domain, DOMAIN_METHODS), (parallel.RankWorker, WORKER_METHODS),
                       (parallel.Scheduler, SCHEDULER_METHODS),
                       (parallel.Transport, TRANSPORT_METHODS)):
        assert all(hasattr(cls, n) for n in names), (cls, names)


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference source tree absent (GPU box)")
    pytest.importorskip("numba")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    return lambda mod: importlib.import_module("hexdg." + mod)


@pytest.mark.parametrize("mod", sorted(NAMES))
def test_signatures_match_reference(ref, mod):
    r = ref(mod)
    o = importlib.import_module("paper_2404_12703_b200." + mod)
    bad = []
    for n in NAMES[mod]:
        if not hasattr(r, n):
            continue
        if not _compatible(getattr(r, n), getattr(o, n)):
            bad.append((n, str(inspect.signature(getattr(r, n))),
                        str(inspect.signature(getattr(o, n)))))
    assert not bad, bad


def test_method_signatures_match_reference(ref):
    from paper_2404_12703_b200 import operator, parallel
    pairs = [(ref("operator").Domain, operator.Domain, DOMAIN_METHODS),
             (ref("parallel").RankWorker, parallel.RankWorker, WORKER_METHODS),
             (ref("parallel").Scheduler, parallel.Scheduler, SCHEDULER_METHODS),
             (ref("parallel").Transport, parallel.Transport, TRANSPORT_METHODS)]
    bad = []
    for rc, oc, names in pairs:
        for n in names:
            if not _compatible(getattr(rc, n), getattr(oc, n)):
                bad.append((oc.__name__, n))
    assert not bad, bad
