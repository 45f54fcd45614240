"""torchrun driver for the multi-GPU tests: run a small TGV case on all ranks and
save rank 0's gathered state. Usage (from the repo root):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29555 tests/mr_driver.py OUT.npz [viscous] [exact] [steps] [N] [mesh]

MRD_RESTART=snap.hdgf resumes from a snapshot; MRD_SNAPSHOT=snap.hdgf writes one at the end.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def case(world, viscous=True, exact=False, steps=3, N=3, mesh=4, prio=True):
    from paper_2404_12703_b200.config import RunConfig
    two_pi = 2 * np.pi
    return RunConfig(testcase="tgv", n=N, mach=0.3, muref=(1.0 / 400.0) if viscous else 0.0,
                     meshx=mesh, meshy=mesh, meshz=mesh, x0=0.0, x1=two_pi, y0=0.0, y1=two_pi,
                     z0=0.0, z1=two_pi, maxsteps=steps, tend=1e9, nranks=world,
                     analyzeinterval=2, priorityscheduling=prio)


def main():
    out = sys.argv[1]
    viscous = sys.argv[2] == "1" if len(sys.argv) > 2 else True
    exact = sys.argv[3] == "1" if len(sys.argv) > 3 else False
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    N = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    mesh = int(sys.argv[6]) if len(sys.argv) > 6 else 4
    prio = sys.argv[7] == "1" if len(sys.argv) > 7 else True
    os.environ["HEXDG_EXACT"] = "1" if exact else "0"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    from paper_2404_12703_b200.parallel import run_distributed
    cfg = case(world, viscous, exact, steps, N, mesh, prio)
    cfg.restartfile = os.environ.get("MRD_RESTART", "")     # resume from an HDGF snapshot
    res = run_distributed(cfg)
    if int(os.environ.get("RANK", "0")) == 0:
        if os.environ.get("MRD_SNAPSHOT"):
            from paper_2404_12703_b200.io import write_snapshot
            write_snapshot(os.environ["MRD_SNAPSHOT"], res.U, res.t, res.alpha)
        keys = sorted(res.series[0])
        np.savez(out, U=res.U, t=res.t, steps=res.steps,
                 traces=res.phase_counts.get("traces", 0),
                 series=np.array([[row[k] for k in keys] for row in res.series]),
                 window=sum(c["window"] for c in res.comm_stats),
                 covered=sum(c["covered"] for c in res.comm_stats),
                 ntrace=len(res.trace))


if __name__ == "__main__":
    main()
