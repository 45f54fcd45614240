"""NVLink evidence for the fused gather + peer-store send kernel, in ONE process on two
GPUs (so ncu may profile it: no multi-rank command under ncu).

    python tools/nvlink_probe.py [rows]            # timing + correctness, JSON line
    ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum \\
        -k regex:peer_send python tools/nvlink_probe.py

hdg_peer_send_rows (the f* / face-viscous sender of the multi-GPU stage) gathers rows
of a cuda:0 array in a permuted order and stores them straight into a landing array
on cuda:1 over NVLink (peer access enabled for the primary contexts), then releases
the landing GPU's flag word. The multi-GPU runs map the neighbour's arrays with
CUDA IPC instead; the kernel and its stores are the same.
"""
import ctypes
import json
import sys

import numpy as np

sys.path.insert(0, ".")


def main():
    import torch
    from paper_2404_12703_b200 import _lib
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
    if torch.cuda.device_count() < 2:
        print(json.dumps({"skipped": "needs 2 GPUs"}))
        return
    lib = _lib.load()
    try:
        rt = ctypes.CDLL("libcudart.so")
    except OSError:
        rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
    for a, b in ((0, 1), (1, 0)):
        assert rt.cudaSetDevice(a) == 0
        rc = rt.cudaDeviceEnablePeerAccess(b, 0)
        assert rc in (0, 704), rc   # 704: already enabled
    torch.cuda.set_device(0)
    d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
    width = 64 * 5                              # one side's f* row at N = 7 (n2 x 5 doubles)
    src = torch.randn((rows, width), dtype=torch.float64, device=d0)
    land = torch.zeros((rows, width), dtype=torch.float64, device=d1)
    flag = torch.zeros(1, dtype=torch.int64, device=d1)
    rng = np.random.default_rng(0)
    dst_rows = rng.permutation(rows).astype(np.int32)
    idx = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=d0)
    nbr, srci, dsti = idx(np.zeros(rows)), idx(np.arange(rows)), idx(dst_rows)
    u64 = lambda v: torch.tensor(np.asarray(v, dtype=np.uint64).view(np.int64), dtype=torch.int64,
                                 device=d0)
    base, flags = u64([land.data_ptr()]), u64([flag.data_ptr()])
    counter = torch.zeros(1, dtype=torch.int32, device=d0)
    epoch = torch.zeros(1, dtype=torch.int64, device=d0)
    s = _lib.stream_ptr()

    def send():
        _lib.check(lib.hdg_peer_send_rows(
            _lib.ptr(src), width, _lib.ptr(nbr), _lib.ptr(srci), _lib.ptr(dsti), rows,
            _lib.ptr(base), _lib.ptr(flags), 1, ctypes.c_void_p(counter.data_ptr()),
            ctypes.c_void_p(epoch.data_ptr()), s), "hdg_peer_send_rows")

    for _ in range(3):
        send()
    torch.cuda.synchronize(d0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        send()
    e1.record()
    torch.cuda.synchronize(d0)
    ms = e0.elapsed_time(e1) / reps
    torch.cuda.synchronize(d1)
    ok = bool(torch.equal(land[torch.as_tensor(dst_rows.astype(np.int64), device=d1)], src.to(d1)))
    nbytes = rows * width * 8
    print(json.dumps({
        "what": "hdg_peer_send_rows: permuted row gather on cuda:0 stored into a cuda:1 array over "
                "NVLink (peer access), + grid-completion flag release",
        "rows": rows, "row_bytes": width * 8, "payload_bytes": nbytes, "ms_per_send": ms,
        "gbs_per_direction": nbytes / (ms * 1e-3) / 1e9,
        "peer_copy_peak_gbs": 770.0, "peak_source": "/opt/skills/guides/B200_PROFILING.md (measured peer copy)",
        "frac": nbytes / (ms * 1e-3) / 1e9 / 770.0,
        "rows_landed_correctly": ok, "flag": int(flag.item()), "epoch": int(epoch.item())}))


if __name__ == "__main__":
    main()
