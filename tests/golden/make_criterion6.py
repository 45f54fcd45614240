"""Acceptance criterion 6 (reference tests/test_acceptance.py:143-161) run by the
REFERENCE itself in the build container (numba, 8 threads, ~15 min):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_criterion6.py

Writes tests/golden/criterion6_reference.json. The reference does NOT meet the
criterion's ">= 90 % of elements with alpha = 0 at t = 10" bar (it reports 0 %);
tests/test_gpu_acceptance.py checks the device run against this record.
"""
import os
import time, numpy as np, json
from hexdg.config import RunConfig
from hexdg.parallel import run_distributed
from hexdg.testcases import TGVSetup
TWO_PI=2*np.pi
setup = TGVSetup(mach=1.25, reynolds=1600.0, version=2)
t0 = setup.T0(RunConfig().gas())
cfg = RunConfig(testcase="tgv", operator="split", nodetype="LGL", x0=0.0, x1=TWO_PI, y0=0.0, y1=TWO_PI, z0=0.0, z1=TWO_PI,
                mach=1.25, reynolds=1600.0, n=7, meshx=8, meshy=8, meshz=8, muref=1.0/1600.0, viscosity="sutherland",
                tref=t0, tgvversion=2, tend=10.0, analyzeinterval=50, shockcapture=True, alphamax=0.5)
w0=time.time()
res = run_distributed(cfg)
out = {"t": res.t, "steps": res.steps, "max_alpha": max(r["max_alpha"] for r in res.series),
       "frac_zero": float(np.mean(res.alpha == 0.0)), "finite": bool(np.isfinite(res.U).all()),
       "series": [(r["t"], r["max_alpha"], r["E_k"]) for r in res.series], "wall": time.time()-w0}
json.dump(out, open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "criterion6_reference.json"), "w"), indent=1)
print(out["t"], out["frac_zero"], out["max_alpha"], out["wall"])
