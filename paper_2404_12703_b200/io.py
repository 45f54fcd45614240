"""On-disk formats of the reference (``src/io.py``), byte-compatible.

* HDGF field snapshots (src/io.py:24-55): little-endian; b"HDGF", uint32
  (version 1, N, nelem, nvar), float64 time, then U in the canonical layout
  (variable fastest, nodes i-fastest, element major) and one float64 blending
  factor per element. ``write_snapshot`` also takes a device tensor and streams
  it through a pinned staging buffer in element chunks, so a 175M-DOF field is
  never duplicated in host memory; ``read_snapshot(..., mmap=True)`` maps it.
* Time-series CSV (src/io.py:58-73): fixed column order, ``repr`` floats, so a
  row round-trips bit for bit.
* Scheduler trace CSV (src/io.py:76-91).
"""

import csv
import struct

import numpy as np

MAGIC = b"HDGF"
FORMAT_VERSION = 1
_HEADER = struct.Struct("<4s4Id")           # magic, version, N, nelem, nvar, time

SERIES_COLUMNS = ["t", "E_k", "eps_S", "eps_D", "dt", "mass", "mom_x",
                  "mom_y", "mom_z", "energy", "max_alpha"]
TRACE_COLUMNS = ["task", "priority", "start", "end", "rank"]


class SnapshotError(ValueError):
    pass


def _is_tensor(a):
    return type(a).__module__.startswith("torch")


def write_snapshot(path, U, time: float, alpha=None, chunk_elems: int = 4096):
    """Write a field snapshot; U has shape (nelem, n1, n1, n1, nvar), numpy or torch."""
    shape = tuple(U.shape)
    if len(shape) != 5 or not (shape[1] == shape[2] == shape[3]):
        raise SnapshotError(f"U must be (nelem, n1, n1, n1, nvar), got {shape}")
    nelem, n1, nvar = shape[0], shape[1], shape[4]
    if alpha is None:
        alpha = np.zeros(nelem)
    alpha = alpha.detach().cpu().numpy() if _is_tensor(alpha) else np.asarray(alpha)
    if alpha.shape != (nelem,):
        raise SnapshotError(f"alpha must have one entry per element, got {alpha.shape}")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, FORMAT_VERSION, n1 - 1, nelem, nvar, float(time)))
        if _is_tensor(U):
            import torch
            src = U.detach().reshape(nelem, -1)
            if src.dtype != torch.float64:
                src = src.to(torch.float64)
            rows = min(chunk_elems, max(nelem, 1))
            stage = torch.empty((rows, src.shape[1]), dtype=torch.float64,
                                pin_memory=src.is_cuda)
            for lo in range(0, nelem, rows):
                hi = min(lo + rows, nelem)
                stage[:hi - lo].copy_(src[lo:hi])
                fh.write(memoryview(stage[:hi - lo].numpy()).cast("B"))
        else:
            fh.write(np.ascontiguousarray(U, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(alpha, dtype="<f8").tobytes())


def read_snapshot(path, mmap: bool = False):
    """Read a snapshot; returns (U, time, alpha)."""
    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
    if len(head) < 4 or head[:4] != MAGIC:
        raise SnapshotError(f"not a snapshot file (magic {head[:4]!r})")
    if len(head) < _HEADER.size:
        raise SnapshotError("truncated snapshot header")
    _, version, N, nelem, nvar, time = _HEADER.unpack(head)
    if version != FORMAT_VERSION:
        raise SnapshotError(f"unsupported snapshot version {version}")
    n1 = N + 1
    count = nelem * n1 ** 3 * nvar
    shape = (nelem, n1, n1, n1, nvar)
    try:
        if mmap:
            U = np.memmap(path, dtype="<f8", mode="r", offset=_HEADER.size, shape=shape)
        else:
            U = np.fromfile(path, dtype="<f8", count=count, offset=_HEADER.size).reshape(shape)
        alpha = np.fromfile(path, dtype="<f8", count=nelem, offset=_HEADER.size + 8 * count)
    except ValueError as exc:
        raise SnapshotError(f"truncated snapshot: {exc}") from exc
    if alpha.size != nelem:
        raise SnapshotError("truncated snapshot: missing blending factors")
    if not mmap:
        U = U.astype(np.float64, copy=False)
    return U, float(time), alpha.astype(np.float64, copy=False)


def write_series_csv(path, series):
    """Analysis rows (dicts) in the canonical column order, repr floats."""
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(SERIES_COLUMNS)
        out.writerows([repr(float(row.get(c, 0.0))) for c in SERIES_COLUMNS] for row in series)


def read_series_csv(path):
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    header = rows[0]
    return [dict(zip(header, map(float, r))) for r in rows[1:]]


def write_trace_csv(path, trace):
    """Trace rows (objects or dicts with task, priority, start, end, rank)."""
    def get(row, k):
        return row[k] if isinstance(row, dict) else getattr(row, k)
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(TRACE_COLUMNS)
        for row in trace:
            out.writerow([get(row, "task"), get(row, "priority"), f"{get(row, 'start'):.9f}",
                          f"{get(row, 'end'):.9f}", get(row, "rank")])


def read_trace_csv(path):
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    return [{"task": t, "priority": int(p), "start": float(s), "end": float(e), "rank": int(r)}
            for t, p, s, e, r in rows[1:]]
