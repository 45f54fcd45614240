"""Multi-rank exchange plan (host logic) -- CPU only, including a world_size-2 gloo run.

Checks the reference's a-priori ordering contract (src/operator.py:587-601,
src/parallel.py:348-377): per neighbour pair, both ends agree on the message
order and length with no metadata, traces go both ways into the slot the
receiver does not own, face viscous fluxes go replica -> primary owner and
surface fluxes primary -> replica owner.
"""

import os

import numpy as np
import pytest

from paper_2404_12703_b200 import mesh as mm
from paper_2404_12703_b200.basis import build_basis
from paper_2404_12703_b200.equations import GasProperties
from paper_2404_12703_b200.exchange import ExchangePlan
from paper_2404_12703_b200.operator import Domain


def _domains(nranks, n=(4, 3, 3), periodic=(True, True, False)):
    m = mm.generate_box_mesh(*n, [(0.0, 1.0)] * 3, periodic)
    m = mm.curve_mesh(mm.random_flips(m, seed=4), 0.03)
    b = build_basis(2, "LGL")
    mm.compute_metrics(m, b)
    parts = mm.partition_sfc(m, nranks)
    er = np.repeat(np.arange(nranks), [p.n_elems for p in parts])
    return m, [Domain(m, b, GasProperties(), p.lo, p.hi, er, p.rank) for p in parts]


@pytest.mark.parametrize("nranks", [2, 3, 5, 8])
def test_plans_pair_up(nranks):
    m, doms = _domains(nranks)
    plans = [ExchangePlan(d) for d in doms]
    for r, (d, p) in enumerate(zip(doms, plans)):
        assert sorted(d.neighbors) == p.nbrs
        for q in p.nbrs:
            dq, pq = doms[q], plans[q]
            # the same global sides, in the same (global id) order, on both ends
            g_r = d.side_global[p.trace_send[q]]
            g_q = dq.side_global[pq.trace_send[r]]
            assert np.array_equal(g_r, g_q)
            assert np.all(np.diff(g_r) > 0)
            # message lengths agree in every phase and direction
            assert p.trace_send[q].size == pq.trace_recv_rows[r].size
            assert p.visc_send_rows[q].size == pq.visc_recv_rows[r].size
            assert p.flux_send_rows[q].size == pq.flux_recv_rows[r].size
            # flux goes from the primary's owner to the replica's owner
            gs = d.side_global[p.flux_send_rows[q]]
            assert np.all((m.side_elem_p[gs] >= d.lo) & (m.side_elem_p[gs] < d.hi))
            gv = d.side_global[(p.visc_send_rows[q] - 1) // 2]
            assert np.all((m.side_elem_r[gv] >= d.lo) & (m.side_elem_r[gv] < d.hi))
            # received traces fill the slot this rank does not own
            rows = p.trace_recv_rows[q]
            side = np.where(rows >= d.ns, rows - d.ns, rows)
            gsd = d.side_global[side]
            own_primary = (m.side_elem_p[gsd] >= d.lo) & (m.side_elem_p[gsd] < d.hi)
            assert np.array_equal(rows >= d.ns, own_primary)


def test_every_partition_side_is_exchanged_once():
    m, doms = _domains(4)
    plans = [ExchangePlan(d) for d in doms]
    cut = set()
    for d, p in zip(doms, plans):
        for q in p.nbrs:
            cut.update(d.side_global[p.flux_send_rows[q]].tolist())
    er = np.repeat(np.arange(4), [d.ne for d in doms])
    inner = np.flatnonzero(m.side_elem_r >= 0)
    expect = set(inner[er[m.side_elem_p[inner]] != er[m.side_elem_r[inner]]].tolist())
    assert cut == expect


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, doms = _domains(world)
        d = doms[rank]
        p = ExchangePlan(d)
        n2 = p.n2

        def trace(gside, role):
            # deterministic fake trace of (global side, role) on (q, p, v)
            return (1000.0 * gside + 10.0 * role + np.arange(n2 * 5)).astype(np.float64)

        own_role = lambda s: 0 if (d.lo <= m.side_elem_p[d.side_global[s]] < d.hi) else 1
        UB = np.zeros((2 * d.ns, n2 * 5))
        sends, recvs = [], []
        for q in p.nbrs:
            buf = np.concatenate([trace(d.side_global[s], own_role(s)) for s in p.trace_send[q]])
            sends.append(dist.P2POp(dist.isend, torch.from_numpy(buf), q))
            rb = torch.zeros(p.trace_recv_rows[q].size * n2 * 5, dtype=torch.float64)
            recvs.append((q, rb))
        reqs = dist.batch_isend_irecv(sends + [dist.P2POp(dist.irecv, t, q) for q, t in recvs])
        for r_ in reqs:
            r_.wait()
        for q, rb in recvs:
            UB[p.trace_recv_rows[q]] = rb.numpy().reshape(-1, n2 * 5)
        ok = True
        for q in p.nbrs:
            for s, row in zip(p.trace_send[q], p.trace_recv_rows[q]):
                ok &= np.array_equal(UB[row], trace(d.side_global[s], 1 - own_role(s)))
        out[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_trace_exchange():
    import torch.multiprocessing as tmp
    mgr = tmp.get_context("spawn").Manager()
    out = mgr.dict()
    port = 29600 + os.getpid() % 200
    tmp.spawn(_gloo_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] and out[1]


def test_overlap_statistics_merges_windows_and_clips_tasks():
    """The overlap measure of the scheduler trace (src/parallel.py:252-271)."""
    from paper_2404_12703_b200.exchange import TraceRow, overlap_statistics
    rows = [TraceRow("elem_ei", 0, 0.0, 2.0, 0), TraceRow("flux_inner", 1, 2.0, 3.0, 0),
            TraceRow("update_ub", 1, 5.0, 6.0, 0)]
    total, covered = overlap_statistics(rows, [(1.0, 2.5), (2.0, 4.0), (5.5, 7.0)])
    assert total == 3.0 + 1.5                  # [1,4] and [5.5,7]
    assert covered == 1.0 + 1.0 + 0.5          # [1,2], [2,3], [5.5,6]
    assert overlap_statistics(rows, []) == (0, 0)
    assert 0.0 <= covered <= total


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_peer_send_lists_deliver_every_row_once(nranks):
    """The peer-memory exchange writes row src of the sender straight into row dst
    of the receiver: simulate the three phases on host arrays of every rank and
    check each receiver row gets exactly the payload the NCCL path delivers."""
    from paper_2404_12703_b200.exchange import peer_send_lists
    m, doms = _domains(nranks)
    plans = [ExchangePlan(d) for d in doms]
    recv = [{r: (p.trace_recv_rows[r], p.visc_recv_rows[r], p.flux_recv_rows[r])
             for r in p.nbrs} for p in plans]
    for phase, sends_of, recv_of in ((0, "trace_send", "trace_recv_rows"),
                                     (1, "visc_send_rows", "visc_recv_rows"),
                                     (2, "flux_send_rows", "flux_recv_rows")):
        land = [np.full(4 * d.ns + 2, -1, dtype=np.int64) for d in doms]
        for me, p in enumerate(plans):
            nbr, src, dst = peer_send_lists(p, {r: recv[r][me] for r in p.nbrs}, phase,
                                            getattr(p, sends_of), me)
            for slot, s_row, d_row in zip(nbr, src, dst):
                r = p.nbrs[slot]
                assert land[r][d_row] == -1, "row written twice"
                land[r][d_row] = doms[me].side_global[s_row % doms[me].ns if phase == 0 else
                                                      (s_row // 2 if phase == 1 else s_row)]
        for me, (d, p) in enumerate(zip(doms, plans)):
            for r in p.nbrs:
                rows = getattr(p, recv_of)[r]
                got = land[me][rows]
                side = rows % d.ns if phase == 0 else (rows // 2 if phase == 1 else rows)
                assert np.array_equal(got, d.side_global[side])
