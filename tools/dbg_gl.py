import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2404_12703_b200.config import RunConfig
from paper_2404_12703_b200.parallel import run_distributed
for nt, op in (("GL", "standard"), ("LGL", "split")):
    cfg = RunConfig(testcase="mms", n=2, nodetype=nt, operator=op, meshx=2, meshy=2, meshz=2,
                    x0=-1.0, x1=1.0, y0=-1.0, y1=1.0, z0=-1.0, z1=1.0, tend=1.0, maxsteps=3,
                    analyzeinterval=1)
    try:
        res = run_distributed(cfg)
        print(nt, "t", res.t, "steps", res.steps, [r["dt"] for r in res.series], flush=True)
    except Exception as e:
        print(nt, "ERR", repr(e), flush=True)
