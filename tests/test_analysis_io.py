"""Analysis partials (oracle restatement pinned to the reference) and the
on-disk formats (byte-compatible with the reference's own files). CPU only."""

import os

import numpy as np

from conftest import GOLDEN, golden


def _analysis_domain(n, curve):
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.mesh import compute_metrics, curve_mesh, generate_box_mesh
    two_pi = 2 * np.pi
    m = generate_box_mesh(2, 2, 2, [(0.0, two_pi)] * 3, (True,) * 3)
    if curve:
        m = curve_mesh(m, curve)
    basis = build_basis(n)
    compute_metrics(m, basis)
    return m, basis


def test_oracle_analysis_partials_bitwise():
    import oracle
    from paper_2404_12703_b200.equations import GasProperties
    from paper_2404_12703_b200.operator import Domain
    from paper_2404_12703_b200.testcases import TGVSetup, reduce_tgv_quantities
    z = golden("analysis_partials")
    m, basis = _analysis_domain(4, 0.05)
    gas = GasProperties(mu_ref=1.0 / 1600.0)
    od = oracle.OracleDomain(Domain(m, basis, gas), basis, gas)
    od.U[...] = z["ns_U"]
    rows = od.analysis_partials(float(z["ns_mu0"]), g=np.ascontiguousarray(z["ns_g"]))
    assert np.array_equal(rows, z["ns_partials"])
    q = reduce_tgv_quantities(rows, TGVSetup(mach=0.3, reynolds=1600.0))
    for k, v in q.items():
        assert v == float(z["ns_q_" + k]), k
    m, basis = _analysis_domain(3, 0.0)
    gas = GasProperties()
    od = oracle.OracleDomain(Domain(m, basis, gas), basis, gas)
    od.U[...] = z["eu_U"]
    assert np.array_equal(od.analysis_partials(0.0), z["eu_partials"])


def test_snapshot_reads_reference_bytes(tmp_path):
    from paper_2404_12703_b200 import io as hio
    U_ref = np.load(os.path.join(GOLDEN, "snapshot_ref_U.npy"))
    U, t, alpha = hio.read_snapshot(os.path.join(GOLDEN, "snapshot_ref.hdgf"))
    assert np.array_equal(U, U_ref) and t == 0.125
    assert np.array_equal(alpha, [0.0, 0.3, 1.0])
    # and writes the same bytes
    out = tmp_path / "s.hdgf"
    hio.write_snapshot(out, U_ref, 0.125, alpha=np.array([0.0, 0.3, 1.0]))
    with open(out, "rb") as a, open(os.path.join(GOLDEN, "snapshot_ref.hdgf"), "rb") as b:
        assert a.read() == b.read()
    Um, tm, am = hio.read_snapshot(out, mmap=True)
    assert np.array_equal(np.asarray(Um), U_ref) and tm == t


def test_snapshot_torch_source_and_errors(tmp_path):
    import pytest
    import torch
    from paper_2404_12703_b200 import io as hio
    rng = np.random.default_rng(3)
    U = rng.standard_normal((37, 4, 4, 4, 5))
    p1, p2 = tmp_path / "a.hdgf", tmp_path / "b.hdgf"
    hio.write_snapshot(p1, U, 1.5)
    hio.write_snapshot(p2, torch.as_tensor(U), 1.5, chunk_elems=8)   # chunked staging
    assert p1.read_bytes() == p2.read_bytes()
    (tmp_path / "bad").write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(hio.SnapshotError):
        hio.read_snapshot(tmp_path / "bad")
    raw = bytearray(p1.read_bytes())
    raw[4] = 9
    (tmp_path / "v9").write_bytes(bytes(raw))
    with pytest.raises(hio.SnapshotError):
        hio.read_snapshot(tmp_path / "v9")
    (tmp_path / "short").write_bytes(p1.read_bytes()[:500])
    with pytest.raises(hio.SnapshotError):
        hio.read_snapshot(tmp_path / "short")
    with pytest.raises(hio.SnapshotError):
        hio.write_snapshot(tmp_path / "x", U, 0.0, alpha=np.zeros(3))


def test_series_csv_matches_reference_bytes(tmp_path):
    from paper_2404_12703_b200 import io as hio
    for tag in ("ns", "eu"):
        ref = os.path.join(GOLDEN, f"series_{tag}.csv")
        rows = hio.read_series_csv(ref)
        out = tmp_path / f"{tag}.csv"
        hio.write_series_csv(out, rows)
        with open(ref, "rb") as fh:
            assert out.read_bytes() == fh.read()
        z = golden("run_series")
        cols = [str(c) for c in z["columns"]]
        for r, row in zip(z[tag + "_series"], rows):
            for c in hio.SERIES_COLUMNS:
                assert row[c] == r[cols.index(c)]


def test_trace_csv_round_trip(tmp_path):
    from paper_2404_12703_b200 import io as hio
    rows = [{"task": "volume", "priority": 0, "start": 0.123456789, "end": 0.5, "rank": 1},
            {"task": "flux_mpi", "priority": 2, "start": 1e-9, "end": 2.0, "rank": 0}]
    p = tmp_path / "trace.csv"
    hio.write_trace_csv(p, rows)
    assert hio.read_trace_csv(p) == rows


def test_restore_snapshot_host_checks(tmp_path):
    """restore_snapshot takes the rank's element rows and the time, and rejects a
    snapshot of another degree or mesh size (host logic only, no kernels)."""
    import numpy as np
    import pytest
    from paper_2404_12703_b200 import mesh as mm
    from paper_2404_12703_b200 import testcases
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.config import RunConfig
    from paper_2404_12703_b200.io import SnapshotError, write_snapshot
    from paper_2404_12703_b200.parallel import (RankWorker, SlotLimiter, Transport,
                                                restore_snapshot)
    cfg = RunConfig(testcase="tgv", n=2, meshx=2, meshy=2, meshz=2, nranks=2,
                    x0=0.0, x1=2 * np.pi, y0=0.0, y1=2 * np.pi, z0=0.0, z1=2 * np.pi)
    m = mm.generate_box_mesh(2, 2, 2, [(0.0, 2 * np.pi)] * 3, (True,) * 3)
    basis = build_basis(2, "LGL")
    mm.compute_metrics(m, basis)
    parts = mm.partition_sfc(m, 2)
    elem_rank = np.repeat([0, 1], [parts[0].hi - parts[0].lo, parts[1].hi - parts[1].lo])
    w = RankWorker(1, m, basis, cfg.gas(), parts[1], elem_rank, cfg, Transport(2),
                   SlotLimiter(1), testcases.build_case(cfg))
    U = np.random.default_rng(0).standard_normal((8, 3, 3, 3, 5))
    write_snapshot(tmp_path / "ok.hdgf", U, 0.625)
    assert restore_snapshot(w, str(tmp_path / "ok.hdgf")) == 0.625
    assert np.array_equal(w.domain.U, U[parts[1].lo:parts[1].hi])
    write_snapshot(tmp_path / "deg.hdgf", np.zeros((8, 4, 4, 4, 5)), 0.0)
    with pytest.raises(SnapshotError, match="does not match N"):
        restore_snapshot(w, str(tmp_path / "deg.hdgf"))
    write_snapshot(tmp_path / "size.hdgf", np.zeros((27, 3, 3, 3, 5)), 0.0)
    with pytest.raises(SnapshotError, match="elements"):
        restore_snapshot(w, str(tmp_path / "size.hdgf"))
