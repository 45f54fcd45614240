"""Element-pass phase times from an E2_TIMING build (A/B diagnostics).

    HEXDG_BUILD_DIR=abtest/timing HEXDG_NVCC_EXTRA=-DE2_TIMING python -m paper_2404_12703_b200.build
    HEXDG_B200_LIB=abtest/timing/libhexdg_b200.so python tools/phase_times.py [c2] [--exact]

Runs a few C2 steps and prints the mean cycles per element of each phase (thread 0
of every CTA; every phase ends at a block-wide barrier, so these are wall phases).
"""
import ctypes
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402


def main():
    import torch
    from paper_2404_12703_b200 import _lib, testcases
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.mesh import compute_metrics, partition_sfc
    from paper_2404_12703_b200.parallel import RankWorker, SlotLimiter, Transport
    name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
    exact = "--exact" in sys.argv
    _, cfg, curved, _ = bench.build_config(name, 1)
    m = bench.build_mesh(cfg, curved)
    basis = build_basis(cfg.n, cfg.nodetype)
    compute_metrics(m, basis)
    w = RankWorker(0, m, basis, cfg.gas(), partition_sfc(m, 1)[0],
                   np.zeros(m.nelem, dtype=np.int64), cfg, Transport(1), SlotLimiter(1),
                   testcases.build_case(cfg), exact=exact)
    w._prepare()
    w.domain.device.upload_state()
    lib = w.domain.device.lib
    out = (ctypes.c_uint64 * 8)()
    for _ in range(2):
        w.step_device()
    torch.cuda.synchronize()
    lib.hdg_debug_phase_cycles(int(exact), out)
    steps = 4
    for _ in range(steps):
        w.step_device()
    torch.cuda.synchronize()
    rc = lib.hdg_debug_phase_cycles(int(exact), out)
    n_elem_passes = steps * w.scheme.stages * m.nelem
    names = ["top (TMA wait)", "P1 prims", "P3 lifting", "P4 volume", "P5 sum", "P2 vstar",
             "P3a lift volume (E2_TIMING2)", "P3b lift surface (E2_TIMING2)"]
    res = {k: out[i] / n_elem_passes for i, k in enumerate(names)}
    res["total"] = sum(res.values())
    print(json.dumps({"config": name, "exact": exact, "rc": rc,
                      "cycles_per_element": {k: round(v, 1) for k, v in res.items()}}))


if __name__ == "__main__":
    main()
