"""Partition-boundary face exchange over NCCL (one process per GPU).

Replaces the reference's in-process ``Transport`` (src/parallel.py:51-112)
and the send/recv tasks of ``_build_rhs`` (:404-499). Payloads keep the
reference's a-priori order -- per neighbour, shared sides sorted by global
side id (src/operator.py:587-601), no index metadata on the wire -- and the
reference's ownership rules, which make results bitwise independent of the
rank count:

* traces: both directions, each rank sends its own trace (UL if primary, else
  UR) and receives the peer's into the slot it does not own (:348-377);
* face viscous fluxes (Navier-Stokes): the replica's owner computes the
  replica-side half of the BR1 interface flux and ships it to the primary's
  owner (this replaces the reference's three gradient-trace messages and the
  lifted-flux message: vstar is recomputed bit-identically from the traces
  on both sides, and only the 4-component face flux crosses the link);
* fluxes: the primary's owner computes f* once and ships it to the replica's
  owner (:480-499), never recomputed.

:class:`ExchangePlan` is pure host logic (index lists + message sizes) and is
tested with the gloo backend on CPU; :class:`NcclExchange` executes it with
device pack/unpack kernels from the C ABI and ``torch.distributed`` NCCL
point-to-point calls, grouped per phase.
"""

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib

PHASE_TRACES = "traces"
PHASE_FACE_VISC = "face-viscous-fluxes"
PHASE_FLUXES = "fluxes"
PRIO_LOW, PRIO_MID, PRIO_TOP = 0, 1, 2      # src/parallel.py:35


@dataclass
class TraceRow:
    """One executed task (src/parallel.py:140-146); times in seconds."""
    task: str
    priority: int
    start: float
    end: float
    rank: int


def overlap_statistics(trace, comm_windows):
    """(communication-window time, part of it covered by executing tasks): the
    windows are merged first, then every task interval is clipped against them
    (the reference's measure, src/parallel.py:252-271)."""
    merged = []
    for a, b in sorted(comm_windows):
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    total = sum(b - a for a, b in merged)
    covered = sum(max(0.0, min(b, row.end) - max(a, row.start))
                  for row in trace for a, b in merged)
    return total, covered


class StreamTracer:
    """Scheduler trace of one rank from CUDA events on its compute stream.

    A task is bracketed by two events; a communication window runs from the
    event recorded when the grouped send/recv is issued to the event recorded
    once the compute stream has passed its wait. Events are read back after
    the caller's per-step synchronisation (:meth:`collect`).
    """

    def __init__(self, torch, rank, max_rows=4000):
        self.torch, self.rank, self.max_rows = torch, rank, max_rows
        self.base = None
        self.pending = []
        self.rows = []
        self.window_total = self.covered = 0.0
        self.kernel_seconds = {}

    def begin(self):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        if self.base is None:
            self.base = ev
        return ev

    def task(self, name, prio, ev0):
        self.pending.append((True, name, prio, ev0, self.begin()))

    def comm(self, phase, ev0):
        self.pending.append((False, phase, PRIO_TOP, ev0, self.begin()))

    def collect(self):
        """Convert the recorded events (stream already synchronised)."""
        rows, wins = [], []
        for is_task, name, prio, e0, e1 in self.pending:
            a = self.base.elapsed_time(e0) * 1e-3
            b = self.base.elapsed_time(e1) * 1e-3
            if is_task:
                rows.append(TraceRow(name, prio, a, b, self.rank))
                self.kernel_seconds[name] = self.kernel_seconds.get(name, 0.0) + (b - a)
            else:
                wins.append((a, b))
        self.pending.clear()
        total, covered = overlap_statistics(rows, wins)
        self.window_total += total
        self.covered += covered
        if len(self.rows) < self.max_rows:
            self.rows.extend(rows)


class ExchangePlan:
    """Per-neighbour index lists of one rank's Domain (host only)."""

    def __init__(self, domain):
        d = domain
        ns, n2 = d.ns, d.n1 * d.n1
        self.n2 = n2
        self.ns = ns
        self.nbrs = sorted(d.neighbors)
        self.trace_send, self.trace_recv_rows = {}, {}
        self.visc_send_rows, self.visc_recv_rows = {}, {}
        self.flux_send_rows, self.flux_recv_rows = {}, {}
        for r in self.nbrs:
            sides = np.asarray(d.neighbors[r]["sides"], dtype=np.int64)
            prim = np.asarray(d.neighbors[r]["is_primary"], dtype=bool)
            # traces: own trace of every shared side; the peer's lands in the slot we do
            # not own: UR (row ns + s of [UL; UR]) when we are primary, else UL (row s)
            self.trace_send[r] = sides
            self.trace_recv_rows[r] = np.where(prim, ns + sides, sides)
            # face viscous fluxes: replica owner -> primary owner, rows 2s+1 of fvface
            self.visc_send_rows[r] = 2 * sides[~prim] + 1
            self.visc_recv_rows[r] = 2 * sides[prim] + 1
            # fluxes: primary owner -> replica owner, rows s of fstar
            self.flux_send_rows[r] = sides[prim]
            self.flux_recv_rows[r] = sides[~prim]

    def message_sizes(self, viscous):
        """Doubles per (neighbour, phase), both directions (for counters/tests)."""
        out = {}
        for r in self.nbrs:
            out[(r, PHASE_TRACES)] = (self.trace_send[r].size * self.n2 * 5,
                                      self.trace_recv_rows[r].size * self.n2 * 5)
            if viscous:
                out[(r, PHASE_FACE_VISC)] = (self.visc_send_rows[r].size * self.n2 * 4,
                                             self.visc_recv_rows[r].size * self.n2 * 4)
            out[(r, PHASE_FLUXES)] = (self.flux_send_rows[r].size * self.n2 * 5,
                                      self.flux_recv_rows[r].size * self.n2 * 5)
        return out


class NcclExchange:
    """Executes the exchange plan of one rank with NCCL point-to-point calls."""

    def __init__(self, rank, world):
        import torch.distributed as dist
        self.dist = dist
        self.rank = rank
        self.world = world
        self.worker = None
        self._row_counts = None
        self.tracer = None      # StreamTracer while RankWorker.run times steps
        self.overlap = True     # cfg.priorityscheduling

    @classmethod
    def from_env(cls, n_ranks):
        import torch
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            local = int(os.environ.get("LOCAL_RANK", "0"))
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        world = dist.get_world_size()
        if world != n_ranks:
            raise ValueError(f"world size {world} != nranks {n_ranks}")
        return cls(dist.get_rank(), world)

    # -- setup ----------------------------------------------------------------
    def attach(self, worker):
        import torch
        self.worker = worker
        self.overlap = bool(worker.cfg.priorityscheduling)
        d = worker.domain
        if d.basis.node_type != "LGL":
            raise NotImplementedError("multi-rank runs use LGL nodes (split or standard form)")
        self.plan = plan = ExchangePlan(d)
        worker._prepare()
        dv = d.device
        self.torch = torch
        dev = dv.dev
        # UL and UR as one (2, ns, n1, n1, 5) block so unpack indexes both with one list
        n1 = d.n1
        self.UB = torch.zeros((2, d.ns, n1, n1, 5), dtype=torch.float64, device=dev)
        dv.UL, dv.UR = self.UB[0], self.UB[1]
        dv._fill_desc()
        it = dv.int_tensor
        self.idx = {}
        self.buf = {}
        for r in plan.nbrs:
            n2 = plan.n2
            self.idx[r] = dict(ts=it(plan.trace_send[r]), tr=it(plan.trace_recv_rows[r]),
                               vs=it(plan.visc_send_rows[r]), vr=it(plan.visc_recv_rows[r]),
                               fs=it(plan.flux_send_rows[r]), fr=it(plan.flux_recv_rows[r]))
            z = lambda n, w: torch.zeros(max(n, 1) * n2 * w, dtype=torch.float64, device=dev)
            self.buf[r] = dict(ts=z(plan.trace_send[r].size, 5), tr=z(plan.trace_recv_rows[r].size, 5),
                               vs=z(plan.visc_send_rows[r].size, 4), vr=z(plan.visc_recv_rows[r].size, 4),
                               fs=z(plan.flux_send_rows[r].size, 5), fr=z(plan.flux_recv_rows[r].size, 5))
        # the primary's owner computes the flux of its partition-boundary sides too
        sides = np.concatenate([d.sides_inner, d.sides_mpi_primary])
        worker.flux_sides = it(sides)
        self.n_flux_sides = int(sides.size)
        self.side_lists = dict(inner=it(d.sides_inner), n_inner=int(d.sides_inner.size),
                               mpi=it(d.sides_mpi_primary), n_mpi=int(d.sides_mpi_primary.size))
        # element passes for overlap (one element per block: N >= 4)
        self.lists = None
        if d.N >= 4 and d.ne > 0 and os.environ.get("HEXDG_SPLIT_PASSES", "1") != "0":
            on_mpi = d.side_is_mpi[d.ef_side].any(axis=1)
            rep_mpi = np.zeros(d.ns, dtype=bool)
            rep_mpi[d.sides_mpi_replica] = True
            on_rep = rep_mpi[d.ef_side].any(axis=1)
            ei, eb = np.flatnonzero(~on_mpi), np.flatnonzero(on_mpi)
            ui, ub = np.flatnonzero(~on_rep), np.flatnonzero(on_rep)
            self.lists = dict(ei=it(ei), n_ei=int(ei.size), eb=it(eb), n_eb=int(eb.size),
                              ui=it(ui), n_ui=int(ui.size), ub=it(ub), n_ub=int(ub.size))

    # -- phases -----------------------------------------------------------------
    # Each phase is split into start (pack on the compute stream, grouped NCCL
    # isend/irecv that waits for the pack) and finish (the compute stream waits for
    # NCCL, then unpacks), so independent work is launched in between and runs
    # while the face data is on the wire (the reference's priority scheduling,
    # src/parallel.py:404-507 / PAPER streams 1-3).
    def _p2p_start(self, sends, recvs, phase):
        ops = [self.dist.P2POp(self.dist.isend, t, p) for p, t in sends if t.numel()] + \
              [self.dist.P2POp(self.dist.irecv, t, p) for p, t in recvs if t.numel()]
        tr = self.worker.transport
        for p, t in sends:
            if t.numel():
                tr.count(self.rank, phase, t.numel() * 8)
        ev = self._tracing() and self.tracer.begin()
        return (self.dist.batch_isend_irecv(ops) if ops else []), ev, phase

    def _p2p_wait(self, handle):
        works, ev, phase = handle
        for w in works:
            w.wait()
        if ev:
            self.tracer.comm(phase, ev)

    def _tracing(self):
        return self.tracer is not None and self.worker.timing_active

    def _task(self, name, prio, fn):
        if not self._tracing():
            fn()
            return
        ev = self.tracer.begin()
        fn()
        self.tracer.task(name, prio, ev)

    def _traces_start(self, U):
        dv = self.worker.domain.device
        lib, s, n2 = dv.lib, dv.sptr(), self.plan.n2
        sends, recvs = [], []
        for r in self.plan.nbrs:
            n = self.plan.trace_send[r].size
            _lib.check(lib.hdg_pack_traces(dv.dptr, _lib.ptr(U), _lib.ptr(self.idx[r]["ts"]), n,
                                           _lib.ptr(self.buf[r]["ts"]), s), "hdg_pack_traces")
            sends.append((r, self.buf[r]["ts"][:n * n2 * 5]))
            recvs.append((r, self.buf[r]["tr"][:self.plan.trace_recv_rows[r].size * n2 * 5]))
        return self._p2p_start(sends, recvs, PHASE_TRACES)

    def _traces_finish(self, works):
        dv = self.worker.domain.device
        lib, s, n2 = dv.lib, dv.sptr(), self.plan.n2
        self._p2p_wait(works)
        for r in self.plan.nbrs:
            n = self.plan.trace_recv_rows[r].size
            _lib.check(lib.hdg_unpack(_lib.ptr(self.buf[r]["tr"]), _lib.ptr(self.idx[r]["tr"]), n,
                                      n2 * 5, _lib.ptr(self.UB), s), "hdg_unpack")

    def exchange_traces(self, U):
        self._traces_finish(self._traces_start(U))

    _SEND = {"vs": "visc_send_rows", "fs": "flux_send_rows"}
    _RECV = {"vr": "visc_recv_rows", "fr": "flux_recv_rows"}

    def _rows_start(self, src, key_s, key_r, width, phase):
        dv = self.worker.domain.device
        lib, s, n2 = dv.lib, dv.sptr(), self.plan.n2
        sends, recvs = [], []
        for r in self.plan.nbrs:
            n_send = getattr(self.plan, self._SEND[key_s])[r].size
            n_recv = getattr(self.plan, self._RECV[key_r])[r].size
            _lib.check(lib.hdg_pack(_lib.ptr(src), _lib.ptr(self.idx[r][key_s]), n_send, n2 * width,
                                    _lib.ptr(self.buf[r][key_s]), s), "hdg_pack")
            sends.append((r, self.buf[r][key_s][:n_send * n2 * width]))
            recvs.append((r, self.buf[r][key_r][:n_recv * n2 * width]))
        return self._p2p_start(sends, recvs, phase)

    def _rows_finish(self, works, dst, key_r, width):
        dv = self.worker.domain.device
        lib, s, n2 = dv.lib, dv.sptr(), self.plan.n2
        self._p2p_wait(works)
        for r in self.plan.nbrs:
            n_recv = getattr(self.plan, self._RECV[key_r])[r].size
            _lib.check(lib.hdg_unpack(_lib.ptr(self.buf[r][key_r]), _lib.ptr(self.idx[r][key_r]),
                                      n_recv, n2 * width, _lib.ptr(dst), s), "hdg_unpack")

    def _stage(self, U, out, mode, t_host, A, B, c, time_dev):
        w = self.worker
        d, dv = w.domain, w.domain.device
        lib, s = dv.lib, dv.sptr()
        prm = ctypes.byref(w.prm)
        visc = bool(w.prm.viscous)
        split = w.split_stage   # element pass -> fluxes -> streaming update
        L = self.lists
        sides = self.side_lists
        run = self._task
        ov = self.overlap       # False: every exchange completes before any work
        ptr = _lib.ptr

        def flux(which, prio):
            run(f"flux_{which}", prio, lambda: _lib.check(lib.hdg_phase_flux(
                dv.dptr, prm, ptr(U), ptr(sides[which]), sides["n_" + which], w.prm.surf_solver,
                s), "hdg_phase_flux"))

        def elem(which, reset, prio):
            run(f"elem_{which}", prio, lambda: _lib.check(lib.hdg_phase_elem_list(
                dv.dptr, prm, ptr(U), ptr(L[which]), L["n_" + which], reset, s),
                "hdg_phase_elem_list"))

        def elem_all():
            run("elem", PRIO_LOW, lambda: _lib.check(lib.hdg_phase_elem(dv.dptr, prm, ptr(U), s),
                                                      "hdg_phase_elem"))

        def update(which, reset, prio):
            run(f"update_{which}", prio, lambda: _lib.check(lib.hdg_phase_update_list(
                dv.dptr, prm, ptr(U), ptr(out), ptr(time_dev), t_host, A, B, c, mode,
                ptr(L[which]), L["n_" + which], reset, s), "hdg_phase_update_list"))

        wk = self._traces_start(U)
        if not ov:
            self._traces_finish(wk)
        if visc and L is not None:
            # interior elements need no halo trace: lift + volume while traces travel
            elem("ei", 1, PRIO_LOW)
            if ov:
                self._traces_finish(wk)
            elem("eb", 0, PRIO_MID)
        elif visc:
            if ov:
                self._traces_finish(wk)
            elem_all()
        else:
            # Euler: the element pass (no lifting) and the inner-side fluxes need no
            # halo trace
            if split:
                elem_all()
            flux("inner", PRIO_MID)
            if ov:
                self._traces_finish(wk)
        if visc:
            wk = self._rows_start(dv.fvface, "vs", "vr", 4, PHASE_FACE_VISC)
            if not ov:
                self._rows_finish(wk, dv.fvface, "vr", 4)
            flux("inner", PRIO_MID)
            if ov:
                self._rows_finish(wk, dv.fvface, "vr", 4)
        flux("mpi", PRIO_TOP)
        wk = self._rows_start(dv.fstar, "fs", "fr", 5, PHASE_FLUXES)
        if not ov:
            self._rows_finish(wk, dv.fstar, "fr", 5)
        if split and L is not None and not w.prm.shock:
            # elements without a partition-boundary replica face update meanwhile
            update("ui", 1, PRIO_LOW)
            if ov:
                self._rows_finish(wk, dv.fstar, "fr", 5)
            update("ub", 0, PRIO_MID)
            return
        if ov:
            self._rows_finish(wk, dv.fstar, "fr", 5)
        fn = lib.hdg_phase_update if split else lib.hdg_phase_volume
        run("update" if split else "volume", PRIO_LOW, lambda: _lib.check(fn(
            dv.dptr, prm, ptr(U), ptr(out), ptr(time_dev), t_host, A, B, c, mode, s),
            "stage volume/update"))

    def rhs(self, worker, U, Ut, t):
        self._stage(U, Ut, _lib.MODE_STORE_UT, t, 0.0, 0.0, 0.0, None)
        return Ut

    def stage(self, worker, U, dU, i, first):
        """``first``: bit 0 first stage, bit 1 (_lib.STAGE_NEXT_DT) fold the next step's
        local dt into the update epilogue (mode flag 64 << 4)."""
        sc = worker.scheme
        mode = _lib.MODE_LSERK_FIRST if (first & 1) else _lib.MODE_LSERK
        if first & _lib.STAGE_NEXT_DT:
            mode |= 64 << 4
        self._stage(U, dU, mode, 0.0, float(sc.A[i]), float(sc.B[i]), float(sc.c[i]),
                    worker.time_dev)

    # -- collectives ------------------------------------------------------------
    def allreduce_dt(self, worker):
        """Global min dt (exact: positive doubles order like int64) and OR of the
        status words (src/parallel.py:567-579, :595-604)."""
        dv = worker.domain.device
        self.dist.all_reduce(dv.dt_bits, op=self.dist.ReduceOp.MIN)
        self.dist.all_reduce(dv.status, op=self.dist.ReduceOp.MAX)

    def barrier(self):
        self.dist.barrier()

    def close(self):
        pass

    def gather_objects(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def max_over_ranks(self, x):
        t = self.torch.tensor([float(x)], dtype=self.torch.float64,
                              device=self.worker.domain.device.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def agree_status(self, status):
        """Status words (BAD_PRIM / BAD_SIDE / NONFINITE / PEER_TIMEOUT) maxed over all
        ranks after a step, so every rank leaves the time loop at the same step with
        the same error instead of one rank raising alone (host array)."""
        t = status.clone()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.cpu().numpy()

    def agree_error(self, err):
        t = self.torch.tensor([1.0 if err is not None else 0.0], device=self.worker.domain.device.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        if err is None and t.item() > 0:
            from .parallel import NumericalFailure
            return NumericalFailure("failure on another rank")
        return err

    def gather_rows(self, rows):
        """Per-element rows (device tensor, leading dim = local ne) of every rank,
        concatenated in rank order = global element order (_gather_rows,
        src/parallel.py:581-591); host array on every rank."""
        torch = self.torch
        rows = rows.contiguous()
        if self._row_counts is None:
            sizes = [None] * self.world
            self.dist.all_gather_object(sizes, int(rows.shape[0]))
            self._row_counts = sizes
        sizes = self._row_counts
        pad = torch.zeros((max(sizes),) + tuple(rows.shape[1:]), dtype=rows.dtype,
                          device=rows.device)
        pad[:rows.shape[0]] = rows
        parts = [torch.empty_like(pad) for _ in sizes]
        self.dist.all_gather(parts, pad)
        return torch.cat([p[:n] for p, n in zip(parts, sizes)]).cpu().numpy()

    def gather_result(self, worker):
        """Rank 0 gets U and alpha in global element order (src/parallel.py:581-591)."""
        torch = self.torch
        d = worker.domain
        dev = d.device.dev
        U_all = self.gather_rows(torch.as_tensor(d.U, device=dev))
        a_all = self.gather_rows(torch.as_tensor(worker.alpha, device=dev))
        wt = self.max_over_ranks(worker.walltime)
        return U_all, a_all, wt


def peer_send_lists(plan, peer_recv_rows, phase, sends, me):
    """Concatenated send list of one phase for the peer-memory exchange:
    (neighbour slot, local source row, destination row in that neighbour's array)
    per message row, neighbours in plan order. peer_recv_rows[r] = rank r's
    (trace, face-viscous, flux) receive rows for messages from this rank, in the
    a-priori message order both ends share (src/operator.py:587-601)."""
    nbr, src, dst = [], [], []
    for slot, r in enumerate(plan.nbrs):
        s_rows = np.asarray(sends[r], dtype=np.int64)
        d_rows = np.asarray(peer_recv_rows[r][phase], dtype=np.int64)
        if s_rows.size != d_rows.size:
            from .parallel import ProtocolError
            raise ProtocolError(f"rank {me}: phase {phase} length mismatch with rank {r}")
        nbr.append(np.full(s_rows.size, slot, dtype=np.int64))
        src.append(s_rows)
        dst.append(d_rows)
    cat = (lambda a: np.concatenate(a) if a else np.zeros(0, np.int64))
    return cat(nbr), cat(src), cat(dst)


class _PeerUnavailable(RuntimeError):
    """Raised on every rank at the same collective point of PeerExchange.attach."""


class PeerExchange(NcclExchange):
    """The same schedule and payloads as :class:`NcclExchange`, with the face data
    moved over NVLink peer memory instead of NCCL point-to-point calls.

    At attach every rank maps its neighbours' landing arrays (the UL/UR halo
    block, fvface, fstar) and flag words with CUDA IPC. A phase start is ONE
    kernel that gathers this rank's rows and stores them straight into the
    neighbours' rows (no staging buffer, no unpack, no communication kernel
    competing for SMs) and, once every block's stores are fenced, releases the
    phase epoch into each neighbour's flag; a phase finish is a one-block
    acquire-spin on this rank's flags (bounded: HDG_STATUS_PEER_TIMEOUT). Every
    rank runs the same phase sequence, so epochs agree without a handshake, and
    the phase dependencies make single landing buffers safe: a neighbour writes
    the next payload of a phase only after it received a later-phase payload
    from this rank that this rank sends after consuming the previous one.
    NCCL stays in use for the once-per-step dt all-reduce.
    """

    PHASES = {PHASE_TRACES: 0, PHASE_FACE_VISC: 1, PHASE_FLUXES: 2}

    @staticmethod
    def available(world):
        import torch
        if int(os.environ.get("LOCAL_WORLD_SIZE", world)) != world or world > 32:
            return False
        n = torch.cuda.device_count()
        if n < world:
            return False
        return all(torch.cuda.can_device_access_peer(a, b)
                   for a in range(world) for b in range(world) if a != b)

    def attach(self, worker):
        super().attach(worker)
        # every rank maps its neighbours or none does: the agreement points inside
        # _attach_peers are collective, so all ranks fall back to NCCL together
        self._nccl_lists = self.lists
        try:
            self._attach_peers(worker)
        except _PeerUnavailable as exc:
            import warnings
            warnings.warn(f"peer-memory exchange unavailable ({exc}); using NCCL send/recv")
            for p in getattr(self, "_mapped", {}).values():
                worker.domain.device.lib.hdg_ipc_close(ctypes.c_void_p(p))
            self._mapped = {}
            self.__class__ = NcclExchange
            self.lists = self._nccl_lists

    def _attach_peers(self, worker):
        torch = self.torch
        d, dv, plan, me = worker.domain, worker.domain.device, self.plan, self.rank
        dev = dv.dev
        self.flags = torch.zeros((3, self.world), dtype=torch.int64, device=dev)
        self.counters = torch.zeros(3, dtype=torch.int32, device=dev)
        # device epoch counters: [0][phase] sends, [1][phase] waits, [2][0] all-reduces
        self.ep = torch.zeros((3, 3), dtype=torch.int64, device=dev)
        # the dt / status all-reduce over peer memory (every rank maps every rank)
        self.red_slots = torch.zeros((2, self.world, 10), dtype=torch.int64, device=dev)
        self.red_flags = torch.zeros(self.world, dtype=torch.int64, device=dev)
        fv = dv.fvface

        def export(t):
            # (cudaIpcMemHandle of the allocation holding t, byte offset of t in it)
            if t is None:
                return None
            if os.environ.get("HEXDG_PEER_FORCE_FAIL") == str(me):   # fallback test hook
                raise _lib.HexdgNativeError("forced export failure")
            h = ctypes.create_string_buffer(64)
            off = ctypes.c_int64()
            _lib.check(dv.lib.hdg_ipc_export(ctypes.c_void_p(t.data_ptr()), h,
                                             ctypes.byref(off)), "hdg_ipc_export")
            return h.raw, int(off.value)

        try:
            mine = {"rows": {r: (plan.trace_recv_rows[r], plan.visc_recv_rows[r],
                                 plan.flux_recv_rows[r]) for r in plan.nbrs},
                    "ipc": {"UB": export(self.UB), "fs": export(dv.fstar), "fv": export(fv),
                            "fl": export(self.flags), "rs": export(self.red_slots),
                            "rf": export(self.red_flags)}}
            note = ""
        except _lib.HexdgNativeError as exc:      # e.g. an allocator without IPC handles
            mine, note = None, str(exc)
        every = self.gather_objects(mine)
        if any(e is None for e in every):
            raise _PeerUnavailable(note or "a rank could not export its buffers")
        torch.cuda.synchronize()
        # map every distinct neighbour block once into THIS device's context
        self._mapped = {}
        self._peers = {}
        note = ""
        try:
            for r in range(self.world):
                if r == me:
                    continue
                self._peers[r] = {}
                for k, v in every[r]["ipc"].items():
                    if v is None:
                        self._peers[r][k] = None
                        continue
                    handle, off = v
                    if handle not in self._mapped:
                        p = ctypes.c_void_p()
                        _lib.check(dv.lib.hdg_ipc_open(handle, ctypes.byref(p)), "hdg_ipc_open")
                        self._mapped[handle] = p.value
                    self._peers[r][k] = self._mapped[handle] + off
        except _lib.HexdgNativeError as exc:
            note = str(exc)
        if not all(self.gather_objects(not note)):
            raise _PeerUnavailable(note or "a rank could not map its neighbours")
        it = dv.int_tensor

        def build(pi, sends, key, width_rows, landing):
            nbr, src, dst = peer_send_lists(plan, {r: every[r]["rows"][me] for r in plan.nbrs},
                                            pi, sends, me)
            base = [self._peers[r][landing] or 0 for r in plan.nbrs]
            flag = [self._peers[r]["fl"] + (pi * self.world + me) * 8 for r in plan.nbrs]
            u64 = (lambda v: torch.tensor(np.asarray(v, dtype=np.uint64).view(np.int64),
                                          dtype=torch.int64, device=dev))
            return dict(nbr=it(nbr), src=it(src), dst=it(dst), n=int(src.size),
                        base=u64(base), flag=u64(flag), width=width_rows,
                        wait=it(np.array([pi * self.world + r for r in plan.nbrs])))

        n2 = plan.n2
        self.peer = {0: build(0, plan.trace_send, "traces", n2 * 5, "UB"),
                     2: build(2, plan.flux_send_rows, "fluxes", n2 * 5, "fs")}
        if fv is not None:
            self.peer[1] = build(1, plan.visc_send_rows, "face-viscous", n2 * 4, "fv")
        # overlap without split passes: one launch per kernel over interior-first
        # orders, the wait for the neighbours' payload fused into the kernel (gate)
        L = self.lists
        self.lists = None
        self.gated = None
        if L is not None:
            cat = lambda a, b: it(np.concatenate([a.cpu().numpy(), b.cpu().numpy()]))
            self.gated = dict(
                elems=cat(L["ei"], L["eb"]), n_e=L["n_ei"] + L["n_eb"], pos_e=L["n_ei"],
                upd=cat(L["ui"], L["ub"]), n_u=L["n_ui"] + L["n_ub"], pos_u=L["n_ui"],
                sides=cat(self.side_lists["inner"], self.side_lists["mpi"]),
                n_s=self.side_lists["n_inner"] + self.side_lists["n_mpi"],
                pos_s=self.side_lists["n_inner"])
        u64 = (lambda v: torch.tensor(np.asarray(v, dtype=np.uint64).view(np.int64),
                                      dtype=torch.int64, device=dev))
        self.red_slot_ptrs = u64([self.red_slots.data_ptr() if r == me else self._peers[r]["rs"]
                                  for r in range(self.world)])
        self.red_flag_ptrs = u64([self.red_flags.data_ptr() if r == me else self._peers[r]["rf"]
                                  for r in range(self.world)])
        self.gather_objects(None)        # every rank mapped its peers before any send

    # -- phases -----------------------------------------------------------------
    def _peer_start(self, pi, phase, src_rows=None, U=None):
        w = self.worker
        dv = w.domain.device
        lib, s = dv.lib, dv.sptr()
        P = self.peer[pi]
        ep = ctypes.c_void_p(self.ep.data_ptr() + 8 * pi)
        ev = self._tracing() and self.tracer.begin()
        ctr = ctypes.c_void_p(self.counters.data_ptr() + 4 * pi)
        n_nbr = len(self.plan.nbrs)
        if pi == 0:
            _lib.check(lib.hdg_peer_send_traces(dv.dptr, _lib.ptr(U), _lib.ptr(P["nbr"]),
                                                _lib.ptr(P["src"]), _lib.ptr(P["dst"]), P["n"],
                                                _lib.ptr(P["base"]), _lib.ptr(P["flag"]), n_nbr,
                                                ctr, ep, s), "hdg_peer_send_traces")
        else:
            _lib.check(lib.hdg_peer_send_rows(_lib.ptr(src_rows), P["width"], _lib.ptr(P["nbr"]),
                                              _lib.ptr(P["src"]), _lib.ptr(P["dst"]), P["n"],
                                              _lib.ptr(P["base"]), _lib.ptr(P["flag"]), n_nbr,
                                              ctr, ep, s), "hdg_peer_send_rows")
        if P["n"]:
            w.transport.count(self.rank, phase, P["n"] * P["width"] * 8)
        return pi, ep, ev, phase

    def _peer_finish(self, handle):
        pi, _, ev, phase = handle
        dv = self.worker.domain.device
        P = self.peer[pi]
        ep = ctypes.c_void_p(self.ep.data_ptr() + 8 * pi)     # the phase's send counter
        _lib.check(dv.lib.hdg_peer_wait(_lib.ptr(self.flags), _lib.ptr(P["wait"]),
                                        len(self.plan.nbrs), ep, _lib.ptr(dv.status), dv.sptr()),
                   "hdg_peer_wait")
        if ev:
            self.tracer.comm(phase, ev)

    def _gate(self, pi, pos):
        g = _lib.HdgGate()
        g.flags = self.flags.data_ptr()
        g.idx = self.peer[pi]["wait"].data_ptr()
        g.n = len(self.plan.nbrs)
        g.pos = pos
        g.epoch = self.ep.data_ptr() + 8 * pi
        return g

    def _stage(self, U, out, mode, t_host, A, B, c, time_dev):
        """Overlapped schedule: the traces travel during the element pass (whose
        boundary elements, listed last, wait for them inside the kernel) and the
        face viscous fluxes during the inner sides' surface fluxes (partition
        sides listed last, same in-kernel wait); the f* exchange is waited for
        explicitly so the update runs over the contiguous element range."""
        w = self.worker
        if not (self.overlap and self.gated is not None and w.split_stage and not w.prm.shock
                and w.prm.viscous):
            return super()._stage(U, out, mode, t_host, A, B, c, time_dev)
        d, dv = w.domain, w.domain.device
        lib, s = dv.lib, dv.sptr()
        prm = ctypes.byref(w.prm)
        ptr = _lib.ptr
        Gd = self.gated
        run = self._task
        h = self._peer_start(0, PHASE_TRACES, U=U)
        g = self._gate(0, Gd["pos_e"])
        run("elem", PRIO_LOW, lambda: _lib.check(lib.hdg_phase_elem_gated(
            dv.dptr, prm, ptr(U), ptr(Gd["elems"]), Gd["n_e"], 1, ctypes.byref(g), s),
            "hdg_phase_elem_gated"))
        if h[2]:
            self.tracer.comm(PHASE_TRACES, h[2])
        # face viscous fluxes: one flux launch over inner ++ partition sides, the
        # blocks of the partition sides wait for the neighbours' halves in-kernel
        h = self._peer_start(1, PHASE_FACE_VISC, src_rows=dv.fvface)
        gs = self._gate(1, Gd["pos_s"])
        run("flux", PRIO_MID, lambda: _lib.check(lib.hdg_phase_flux_gated(
            dv.dptr, prm, ptr(U), ptr(Gd["sides"]), Gd["n_s"], w.prm.surf_solver,
            ctypes.byref(gs), s), "hdg_phase_flux_gated"))
        if h[2]:
            self.tracer.comm(PHASE_FACE_VISC, h[2])
        h = self._peer_start(2, PHASE_FLUXES, src_rows=dv.fstar)
        self._peer_finish(h)
        run("update", PRIO_LOW, lambda: _lib.check(lib.hdg_phase_update(
            dv.dptr, prm, ptr(U), ptr(out), ptr(time_dev), t_host, A, B, c, mode, s),
            "hdg_phase_update"))

    def close(self):
        """Unmap the neighbours' arrays once every rank is done with them."""
        if getattr(self, "_mapped", None):
            self.torch.cuda.synchronize()
            self.gather_objects(None)
            lib = self.worker.domain.device.lib
            for p in self._mapped.values():
                lib.hdg_ipc_close(ctypes.c_void_p(p))
            self._mapped = {}
            self.gather_objects(None)

    def allreduce_dt(self, worker):
        """Min dt bits / max status words over all ranks through peer memory:
        one kernel, no NCCL call, so a whole step is capturable in a CUDA graph."""
        dv = worker.domain.device
        _lib.check(dv.lib.hdg_peer_allreduce_dt(
            dv.dptr, _lib.ptr(self.red_slot_ptrs), _lib.ptr(self.red_flag_ptrs),
            _lib.ptr(self.red_slots), _lib.ptr(self.red_flags), self.rank, self.world,
            ctypes.c_void_p(self.ep.data_ptr() + 8 * 6), dv.sptr()), "hdg_peer_allreduce_dt")

    def _traces_start(self, U):
        return self._peer_start(0, PHASE_TRACES, U=U)

    def _traces_finish(self, works):
        self._peer_finish(works)

    def _rows_start(self, src, key_s, key_r, width, phase):
        return self._peer_start(1 if key_s == "vs" else 2, phase, src_rows=src)

    def _rows_finish(self, works, dst, key_r, width):
        self._peer_finish(works)


def make_exchange(n_ranks):
    """The multi-rank exchange: NVLink peer memory when every rank of the job is
    on this node with peer access (measured 7% faster than NCCL send/recv at 4
    GPUs); HEXDG_EXCHANGE=nccl forces NCCL point-to-point."""
    comm = NcclExchange.from_env(n_ranks)
    mode = os.environ.get("HEXDG_EXCHANGE", "peer")
    if mode == "peer" and PeerExchange.available(n_ranks):
        comm.__class__ = PeerExchange
    return comm
