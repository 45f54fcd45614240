"""Multi-GPU runs over NCCL are bitwise identical to one GPU (the reference's
headline rank-invariance property, tests/test_parallel.py:110-117 and
tests/test_acceptance.py:99-114). Needs >= 2 visible GPUs."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _run(tmp_path, nproc, viscous, exact, steps=3, N=3, mesh=4, prio=True, exchange="peer",
         env_extra=None):
    out = tmp_path / f"U_{nproc}_{int(viscous)}_{int(exact)}_{N}_{int(prio)}_{exchange}.npz"
    if nproc == 1:
        cmd = [sys.executable, os.path.join(ROOT, "tests", "mr_driver.py")]
    else:
        port = 29500 + (os.getpid() * 7 + nproc) % 400
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", str(nproc),
               "--master-addr", "127.0.0.1", "--master-port", str(port),
               os.path.join(ROOT, "tests", "mr_driver.py")]
    cmd += [str(out), str(int(viscous)), str(int(exact)), str(steps), str(N), str(mesh),
            str(int(prio))]
    env = dict(os.environ, HEXDG_EXCHANGE=exchange, **(env_extra or {}))
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    return dict(np.load(out))


@pytest.mark.parametrize("viscous", [True, False], ids=["ns", "euler"])
def test_two_gpus_bitwise_equal_one(tmp_path, viscous):
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    one = _run(tmp_path, 1, viscous, False)
    two = _run(tmp_path, 2, viscous, False)
    assert one["steps"] == two["steps"] == 3
    assert np.array_equal(one["U"], two["U"])
    assert float(one["t"]) == float(two["t"])
    assert int(two["traces"]) > 0
    # analysis rows (every 2 steps + the end) gathered in global element order
    assert np.array_equal(one["series"], two["series"])


@pytest.mark.parametrize("viscous", [True, False], ids=["ns", "euler"])
def test_two_gpus_overlapped_passes_bitwise(tmp_path, viscous):
    """N >= 4 takes the overlapped path (interior / boundary element passes)."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    one = _run(tmp_path, 1, viscous, False, steps=2, N=4, mesh=4)
    two = _run(tmp_path, 2, viscous, False, steps=2, N=4, mesh=4)
    assert np.array_equal(one["U"], two["U"])


def test_four_gpus_uneven_partition_exact(tmp_path):
    if _ngpus() < 4:
        pytest.skip("needs 4 GPUs")
    one = _run(tmp_path, 1, True, True, steps=2, mesh=3)
    four = _run(tmp_path, 4, True, True, steps=2, mesh=3)
    assert np.array_equal(one["U"], four["U"])
    assert np.array_equal(one["series"], four["series"])


def test_priority_scheduling_improves_overlap(tmp_path):
    """Acceptance criterion 10 (tests/test_acceptance.py:226-239): the fraction of
    the communication windows covered by kernel work is larger with the
    overlapped schedule than with every exchange completing before any work;
    both schedules give the same field."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    on = _run(tmp_path, 2, True, False, steps=4, N=4, mesh=6, prio=True)
    off = _run(tmp_path, 2, True, False, steps=4, N=4, mesh=6, prio=False)
    assert np.array_equal(on["U"], off["U"])
    assert int(on["ntrace"]) > 0
    for r in (on, off):
        assert 0.0 < float(r["window"]) and 0.0 <= float(r["covered"]) <= float(r["window"]) * (1 + 1e-9)
    frac_on = float(on["covered"]) / float(on["window"])
    frac_off = float(off["covered"]) / float(off["window"])
    assert frac_on > frac_off, (frac_on, frac_off)


@pytest.mark.parametrize("N", [3, 4])
def test_two_gpus_nccl_exchange_bitwise(tmp_path, N):
    """The NCCL point-to-point exchange (HEXDG_EXCHANGE=nccl, the fallback when the
    ranks have no NVLink peer access) gives the same bits as the peer-memory one."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    a = _run(tmp_path, 2, True, False, steps=2, N=N, mesh=4, exchange="nccl")
    b = _run(tmp_path, 2, True, False, steps=2, N=N, mesh=4, exchange="peer")
    assert np.array_equal(a["U"], b["U"])
    assert np.array_equal(a["series"], b["series"])


def test_peer_exchange_falls_back_to_nccl_together(tmp_path):
    """If one rank cannot export its buffers for CUDA IPC, every rank switches to
    NCCL at the same collective point (no hang) and the run is unchanged."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    (tmp_path / "a").mkdir()
    (tmp_path / "b").mkdir()
    ref = _run(tmp_path / "a", 2, True, False, steps=2, N=4, mesh=4)
    fb = _run(tmp_path / "b", 2, True, False, steps=2, N=4, mesh=4,
              env_extra={"HEXDG_PEER_FORCE_FAIL": "1"})
    assert np.array_equal(ref["U"], fb["U"])


def test_restart_on_two_gpus_from_one_gpu_snapshot(tmp_path):
    """A 1-GPU snapshot after 3 steps resumed on 2 GPUs for 3 more steps equals the
    uninterrupted 6-step 1-GPU run bit for bit (resume + rank invariance)."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    snap = str(tmp_path / "three.hdgf")
    for sub in ("full", "half", "res"):
        (tmp_path / sub).mkdir()
    full = _run(tmp_path / "full", 1, True, False, steps=6)
    _run(tmp_path / "half", 1, True, False, steps=3, env_extra={"MRD_SNAPSHOT": snap})
    res = _run(tmp_path / "res", 2, True, False, steps=3, env_extra={"MRD_RESTART": snap})
    assert float(res["t"]) == float(full["t"])
    assert np.array_equal(res["U"], full["U"])
