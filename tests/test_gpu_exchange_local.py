"""Multi-rank exchange kernels on ONE GPU (so the driver's 1-GPU test run exercises
them): two ranks in one process, each a RankWorker on its SFC partition, with the
NCCL point-to-point transport replaced by an in-process mailbox (host threads, one
per rank, enqueue on the same stream; no kernel ever waits on another kernel, so
nothing can hang the device). The face-data path -- hdg_pack_traces / hdg_pack /
hdg_unpack in the a-priori neighbour order (reference src/parallel.py:348-395),
the interior / boundary element passes and the primary-owner flux rule -- must give
the single-rank result bit for bit. The peer-memory send kernels are checked for
their row placement and their grid-completion epoch (the block counter returns to 0
after every launch)."""

import ctypes
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _Mailbox:
    def __init__(self):
        self.cond = threading.Condition()
        self.box = {}

    def post(self, key, t):
        with self.cond:
            self.box.setdefault(key, []).append(t)
            self.cond.notify_all()

    def take(self, key, timeout=60.0):
        with self.cond:
            ok = self.cond.wait_for(lambda: self.box.get(key), timeout=timeout)
            if not ok:
                raise TimeoutError(f"no message {key}")
            return self.box[key].pop(0)


def _local_exchange_class():
    from paper_2404_12703_b200.exchange import NcclExchange

    class LocalExchange(NcclExchange):
        """NcclExchange with the NCCL calls replaced by device copies through a mailbox."""

        def __init__(self, rank, world, mailbox):
            self.rank, self.world, self.mail = rank, world, mailbox
            self.worker = None
            self._row_counts = None
            self.tracer = None
            self.overlap = True
            self.seq = {}

        def _p2p_start(self, sends, recvs, phase):
            n = self.seq.get(phase, 0)
            self.seq[phase] = n + 1
            for p, t in sends:
                if t.numel():
                    self.worker.transport.count(self.rank, phase, t.numel() * 8)
                    self.mail.post((self.rank, p, phase, n), t.clone())
            return [(p, t, (p, self.rank, phase, n)) for p, t in recvs if t.numel()], None, phase

        def _p2p_wait(self, handle):
            works, _, _ = handle
            for _, t, key in works:
                t.copy_(self.mail.take(key))

    return LocalExchange


def _workers(cfg, mesh, n_ranks, comm_factory=None, exact=False):
    from paper_2404_12703_b200 import testcases
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.mesh import compute_metrics, partition_sfc
    from paper_2404_12703_b200.parallel import RankWorker, SlotLimiter, Transport
    basis = build_basis(cfg.n, cfg.nodetype)
    compute_metrics(mesh, basis)
    parts = partition_sfc(mesh, n_ranks)
    elem_rank = np.repeat(np.arange(n_ranks), [p.n_elems for p in parts])
    ws = []
    for r in range(n_ranks):
        comm = comm_factory(r) if comm_factory else None
        w = RankWorker(r, mesh, basis, cfg.gas(), parts[r], elem_rank, cfg, Transport(n_ranks),
                       SlotLimiter(1), testcases.build_case(cfg), comm=comm, exact=exact)
        if comm is not None:
            comm.attach(w)
        ws.append(w)
    return ws


def _steps(w, dts):
    w._prepare()
    dv = w.domain.device
    dv.upload_state()
    t = 0.0
    for dt in dts:
        w.time_dev[0], w.time_dev[1] = t, float(dt)
        for i in range(w.scheme.stages):
            w.stage_device(dv.U, w.rk_work, i, i == 0)
        t += float(dt)


@pytest.mark.parametrize("viscous,n,shock", [(True, 4, False), (False, 5, False),
                                             (True, 5, True), (True, 7, False)],
                         ids=["ns-n4", "euler-n5", "ns-n5-fv", "ns-n7"])
def test_two_ranks_on_one_gpu_bitwise_equal_one(gpu, viscous, n, shock):
    from paper_2404_12703_b200 import mesh as mm
    from paper_2404_12703_b200.config import RunConfig
    two_pi = 2 * np.pi
    kw = dict(shockcapture=True, indicator="constant", alphaconst=0.3) if shock else {}
    cfg = RunConfig(testcase="tgv", n=n, mach=0.3, muref=(1.0 / 1600.0) if viscous else 0.0,
                    meshx=4, meshy=4, meshz=4, x0=0.0, x1=two_pi, y0=0.0, y1=two_pi, z0=0.0,
                    z1=two_pi, tend=1e9, **kw)

    def mesh():
        return mm.curve_mesh(mm.random_flips(mm.generate_box_mesh(
            4, 4, 4, [(0.0, two_pi)] * 3, (True,) * 3), seed=3), 0.04)
    dts = [2e-3, 1.9e-3, 2.1e-3]
    (single,) = _workers(cfg, mesh(), 1)
    _steps(single, dts)
    ref = single.domain.device.U.cpu().numpy()

    mail = _Mailbox()
    Local = _local_exchange_class()
    ws = _workers(cfg, mesh(), 2, comm_factory=lambda r: Local(r, 2, mail))
    assert all(w.domain.sides_mpi.size for w in ws)      # the partition has halo sides
    errs = []

    def run(w):
        try:
            _steps(w, dts)
        except BaseException as exc:   # noqa: BLE001
            errs.append(exc)
    th = [threading.Thread(target=run, args=(w,)) for w in ws]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    assert not errs, errs
    import torch
    torch.cuda.synchronize()
    got = np.concatenate([w.domain.device.U.cpu().numpy() for w in ws])
    assert np.array_equal(got, ref), float(np.max(np.abs(got - ref)))
    sent = sum(int(w.transport.bytes_sent.sum()) for w in ws)
    assert sent > 0


def test_peer_send_rows_places_rows_and_resets_block_counter(gpu):
    """hdg_peer_send_rows into a local landing array (the IPC-mapped neighbour array's
    stand-in): rows land at their destination rows, the epoch advances by one per
    launch and reaches the neighbour flag, and the grid-completion block counter is
    back at 0 after every launch (it never grows, so it never wraps)."""
    import torch
    from paper_2404_12703_b200 import _lib
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    width, n, n_land = 40, 3000, 4000
    src = torch.randn((n, width), dtype=torch.float64, device=dev)
    land = torch.zeros((n_land, width), dtype=torch.float64, device=dev)
    rng = np.random.default_rng(0)
    dst_rows = rng.permutation(n_land)[:n].astype(np.int32)
    idx = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=dev)
    nbr, srci, dsti = idx(np.zeros(n)), idx(np.arange(n)), idx(dst_rows)
    flag = torch.zeros(1, dtype=torch.int64, device=dev)
    u64 = lambda v: torch.tensor(np.asarray(v, dtype=np.uint64).view(np.int64),
                                 dtype=torch.int64, device=dev)
    base, flags = u64([land.data_ptr()]), u64([flag.data_ptr()])
    counter = torch.zeros(1, dtype=torch.int32, device=dev)
    epoch = torch.zeros(1, dtype=torch.int64, device=dev)
    for k in range(1, 6):
        _lib.check(lib.hdg_peer_send_rows(
            _lib.ptr(src), width, _lib.ptr(nbr), _lib.ptr(srci), _lib.ptr(dsti), n,
            _lib.ptr(base), _lib.ptr(flags), 1, ctypes.c_void_p(counter.data_ptr()),
            ctypes.c_void_p(epoch.data_ptr()), _lib.stream_ptr()), "hdg_peer_send_rows")
        torch.cuda.synchronize()
        assert int(counter.item()) == 0
        assert int(epoch.item()) == k and int(flag.item()) == k
    assert torch.equal(land[torch.as_tensor(dst_rows.astype(np.int64), device=dev)], src)
