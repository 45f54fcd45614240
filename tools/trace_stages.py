"""Scheduler trace of a short multi-GPU run (diagnostics, not a test).

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        tools/trace_stages.py OUT.csv [config] [steps]

Runs ``run_distributed`` on a bench configuration and writes every rank's task
rows (CUDA-event intervals of the kernels of each stage, seconds) with the
reference's trace CSV format; prints the overlap statistics.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    out = sys.argv[1]
    name = sys.argv[2] if len(sys.argv) > 2 else "c2"
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    import bench
    from paper_2404_12703_b200 import io as hio
    from paper_2404_12703_b200.parallel import run_distributed
    world = int(os.environ.get("WORLD_SIZE", "1"))
    _, cfg, curved, _ = bench.build_config(name, world)
    cfg.maxsteps = steps
    mesh = bench.build_mesh(cfg, curved)
    res = run_distributed(cfg, mesh=mesh)
    if int(os.environ.get("RANK", "0")) == 0:
        hio.write_trace_csv(out, res.trace)
        for r, c in enumerate(res.comm_stats):
            print(f"rank {r}: comm window {c['window'] * 1e3:.3f} ms, covered "
                  f"{c['covered'] * 1e3:.3f} ms ({c['covered'] / max(c['window'], 1e-30):.1%})")
        print("walltime per step", res.walltime / max(res.steps, 1))


if __name__ == "__main__":
    main()
