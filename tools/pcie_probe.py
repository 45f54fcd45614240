"""Host<->device copy bandwidth for the e2e leg: default pinned vs NUMA-local pinned
buffers, one direction at a time and full duplex (two copy streams). Diagnostic only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import gpu_local_cpus, pinned_near_gpu  # noqa: E402


def timed(fn, reps=5):
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s0.record()
    for _ in range(reps):
        fn()
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) / reps


def main():
    dev = torch.device("cuda:0")
    n = 671088640 // 8
    d_a = torch.empty(n, dtype=torch.float64, device=dev)
    d_b = torch.empty(n, dtype=torch.float64, device=dev)
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    out = {"cpu_count": os.cpu_count(), "gpu_local_cpus": len(gpu_local_cpus(dev) or ())}
    for name in ("default", "numa_local"):
        if name == "default":
            h_a = torch.zeros(n, dtype=torch.float64, pin_memory=True)
            h_b = torch.zeros(n, dtype=torch.float64, pin_memory=True)
        else:
            h_a, _ = pinned_near_gpu((n,), dev)
            h_b, _ = pinned_near_gpu((n,), dev)
        gb = n * 8 / 1e9

        def h2d():
            d_a.copy_(h_a, non_blocking=True)

        def d2h():
            h_b.copy_(d_b, non_blocking=True)

        def duplex():
            cur = torch.cuda.current_stream()
            up.wait_stream(cur)
            down.wait_stream(cur)
            with torch.cuda.stream(up):
                d_a.copy_(h_a, non_blocking=True)
            with torch.cuda.stream(down):
                h_b.copy_(d_b, non_blocking=True)
            cur.wait_stream(up)
            cur.wait_stream(down)

        out[name] = {"h2d_gbs": gb / (timed(h2d) * 1e-3), "d2h_gbs": gb / (timed(d2h) * 1e-3),
                     "duplex_gbs_each": gb / (timed(duplex) * 1e-3)}
        del h_a, h_b
    print(json.dumps(out))


if __name__ == "__main__":
    main()
