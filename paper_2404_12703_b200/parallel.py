"""Rank runtime: the time-derivative call, the device time loop, multi-rank driver.

Mirror of ``hexdg.parallel`` (reference ``src/parallel.py``). One process
(rank) per GPU. The reference's per-stage task DAG + priority scheduler
(:151-249, :399-517) becomes a fixed sequence of stream-ordered kernels
(lift -> flux -> element kernel with the fused LSERK update); the in-process
``Transport`` (:51-112) becomes NCCL point-to-point exchanges of face data in
the reference's a-priori order (see :mod:`.exchange`). A whole RK step is
captured once in a CUDA graph (:class:`Stepper`).
"""

import ctypes
import os
import threading
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import testcases
from .basis import build_basis
from .config import RunConfig
from .equations import RIEMANN_LLF_SPLIT, RIEMANN_SOLVERS, AdmissibilityError
from .mesh import Mesh, compute_metrics, curve_mesh, generate_box_mesh, load_mesh_cache, \
    partition_sfc
from .operator import NVAR, Domain
from .shock import INDICATOR_CONSTANT, INDICATOR_HENNEMANN, ShockConfig, \
    subcell_interface_metrics
from .timedisc import get_scheme

from .exchange import TraceRow, overlap_statistics  # noqa: E402,F401 (reference import path)

PRIO_LOW, PRIO_MID, PRIO_TOP = 0, 1, 2
PHASE_TRACES = "traces"
PHASE_FLUXES = "fluxes"
PHASE_LIFT_FLUXES = "lifted-fluxes"
PHASE_LIFT_TRACES = "lifted-traces"


class ProtocolError(RuntimeError):
    pass


class NumericalFailure(RuntimeError):
    """The solution left the admissible set (NaN/Inf or negative density)."""


class Transport:
    """In-process FIFO channels keyed by (src, dst, phase) (src/parallel.py:51-112).

    The device runtime moves face data over NVLink peer memory / NCCL (one process
    per GPU, :mod:`.exchange`), not through this object; it carries ``n_ranks``,
    the message/byte counters of those exchanges, and the reference's host message
    API (``send``/``poll``/``wait``/``wait_any``/``abort``) used by
    :class:`Scheduler` task graphs and host-side drivers.
    """

    def __init__(self, n_ranks: int):
        self.n_ranks = n_ranks
        self._cond = threading.Condition()
        self._queues = {}
        self._aborted = None
        self.bytes_sent = np.zeros(n_ranks, dtype=np.int64)
        self.messages_sent = np.zeros(n_ranks, dtype=np.int64)
        self.phase_counts = {}
        self.phase_bytes = {}

    def count(self, src, phase, nbytes):
        """Account one device-side message (the exchange layer calls this)."""
        with self._cond:
            self.bytes_sent[src] += nbytes
            self.messages_sent[src] += 1
            self.phase_counts[phase] = self.phase_counts.get(phase, 0) + 1
            self.phase_bytes[phase] = self.phase_bytes.get(phase, 0) + nbytes

    def send(self, src: int, dst: int, phase: str, payload):
        buf = np.array(payload, dtype=np.float64, copy=True)
        with self._cond:
            self._queues.setdefault((src, dst, phase), deque()).append((buf, time.perf_counter()))
            self.bytes_sent[src] += buf.nbytes
            self.messages_sent[src] += 1
            self.phase_counts[phase] = self.phase_counts.get(phase, 0) + 1
            self.phase_bytes[phase] = self.phase_bytes.get(phase, 0) + buf.nbytes
            self._cond.notify_all()

    def _check(self):
        if self._aborted is not None:
            raise ProtocolError(f"transport aborted: {self._aborted}")

    def poll(self, src: int, dst: int, phase: str):
        """Non-blocking receive: (payload, arrival time) or None."""
        with self._cond:
            self._check()
            q = self._queues.get((src, dst, phase))
            return q.popleft() if q else None

    def wait(self, src: int, dst: int, phase: str):
        """Blocking receive."""
        with self._cond:
            while True:
                self._check()
                q = self._queues.get((src, dst, phase))
                if q:
                    return q.popleft()
                self._cond.wait(timeout=1.0)

    def wait_any(self, probes):
        """Block until any probe() is true (probes must not consume)."""
        with self._cond:
            while True:
                self._check()
                if any(p() for p in probes):
                    return
                self._cond.wait(timeout=1.0)

    def has_message(self, src: int, dst: int, phase: str) -> bool:
        return bool(self._queues.get((src, dst, phase)))

    def abort(self, reason: str):
        with self._cond:
            if self._aborted is None:
                self._aborted = reason
            self._cond.notify_all()


class SlotLimiter:
    """Caps concurrently active ranks of one process (src/parallel.py:115-129).
    Device ranks are processes (one per GPU), so the production path never blocks here."""

    def __init__(self, slots: int):
        self.slots = slots
        self._sem = threading.Semaphore(max(1, slots))

    def acquire(self):
        self._sem.acquire()

    def release(self):
        self._sem.release()


@dataclass
class Task:
    name: str
    fn: object
    deps: tuple = ()
    priority: int = PRIO_LOW
    poll: object = None     # receive tasks: callable -> bool, message available
    order: int = 0


class Scheduler:
    """Host task-graph executor of the reference (src/parallel.py:151-249).

    With priorities enabled, ready tasks run highest priority first, FIFO within a
    class, and a receive task becomes ready only once its message arrived, so
    lower-priority work fills communication latency; disabled, tasks run in
    insertion order and receives block in place. On the device path the same
    policy is realised by stream order (:mod:`.exchange`: boundary work first,
    interior work while the exchange is in flight), and :class:`StreamTracer`
    records the equivalent ``TraceRow``s from CUDA events.
    """

    def __init__(self, rank: int, transport: Transport, limiter: SlotLimiter,
                 priorities_enabled: bool = True):
        self.rank = rank
        self.transport = transport
        self.limiter = limiter
        self.enabled = priorities_enabled
        self.tasks = []
        self.trace = []
        self.comm_windows = []
        self.blocked_time = 0.0

    def add(self, name, fn, deps=(), priority=PRIO_LOW, poll=None):
        self.tasks.append(Task(name, fn, tuple(deps), priority, poll, order=len(self.tasks)))

    def _validate(self):
        known = {t.name: t for t in self.tasks}
        colour = {}

        def visit(t):
            c = colour.get(t.name)
            if c == 1:
                raise ProtocolError(f"task dependency cycle at {t.name!r}")
            if c == 2:
                return
            colour[t.name] = 1
            for d in t.deps:
                if d not in known:
                    raise ProtocolError(f"task {t.name!r} depends on unknown {d!r}")
                visit(known[d])
            colour[t.name] = 2

        for t in self.tasks:
            visit(t)

    def _execute(self, t, posted):
        start = time.perf_counter()
        t.fn()
        end = time.perf_counter()
        self.trace.append(TraceRow(t.name, t.priority, start, end, self.rank))
        if t.poll is not None:
            self.comm_windows.append((posted, end))

    def _block(self, probes):
        start = time.perf_counter()
        self.limiter.release()
        try:
            self.transport.wait_any(probes)
        finally:
            self.limiter.acquire()
        self.blocked_time += time.perf_counter() - start

    def run(self):
        self._validate()
        posted = time.perf_counter()    # receives are posted when the graph starts
        if not self.enabled:
            for t in self.tasks:
                if t.poll is not None and not t.poll():
                    self._block([t.poll])
                self._execute(t, posted)
            return self.trace
        done = set()
        pending = list(self.tasks)
        while pending:
            runnable = [t for t in pending if all(d in done for d in t.deps)]
            ready = [t for t in runnable if t.poll is None or t.poll()]
            if ready:
                t = min(ready, key=lambda x: (-x.priority, x.order))
                self._execute(t, posted)
                done.add(t.name)
                pending.remove(t)
            elif runnable:
                self._block([t.poll for t in runnable])
            else:
                raise ProtocolError(f"rank {self.rank}: no runnable task; "
                                    f"pending {[t.name for t in pending]}")
        return self.trace


@dataclass
class RunResult:
    U: np.ndarray = None
    alpha: np.ndarray = None
    t: float = 0.0
    steps: int = 0
    series: list = field(default_factory=list)
    walltime: float = 0.0
    n_ranks: int = 1
    n_dof: int = 0
    rk_stages: int = 0
    kernel_seconds: list = field(default_factory=list)
    rhs_seconds: list = field(default_factory=list)
    comm_stats: list = field(default_factory=list)
    message_counts: np.ndarray = None
    bytes_sent: np.ndarray = None
    phase_counts: dict = field(default_factory=dict)
    phase_bytes: dict = field(default_factory=dict)
    trace: list = field(default_factory=list)


class RankWorker:
    """One rank: local domain, device state, the rhs, the time loop (src/parallel.py:298-667)."""

    def __init__(self, rank, mesh, basis, gas, partition, elem_rank, cfg: RunConfig,
                 transport: Transport, limiter: SlotLimiter, case, comm=None, exact=None):
        self.rank = rank
        self.cfg = cfg
        self.transport = transport
        self.limiter = limiter
        self.n_ranks = transport.n_ranks
        self.comm = comm
        self.exact = bool(int(os.environ.get("HEXDG_EXACT", "0"))) if exact is None else exact
        self.domain = Domain(mesh, basis, gas, partition.lo, partition.hi, elem_rank, rank)
        self.n_elem_global = mesh.nelem
        self.domain.exact = self.exact
        self.split = cfg.operator == "split"
        self.solver_id = RIEMANN_SOLVERS[cfg.riemann]
        self.surf_solver_id = RIEMANN_LLF_SPLIT \
            if (self.split and cfg.riemann == "llf") else self.solver_id   # :311-314
        self.scheme = get_scheme(cfg.rkscheme)
        self.init_fn, bc_states, self.source, self.case_setup = case
        if bc_states is not None:
            self.domain.bc_states = bc_states
        self.shock = ShockConfig(
            enabled=cfg.shockcapture, alpha_max=cfg.alphamax, alpha_min=cfg.alphamin,
            indicator=INDICATOR_CONSTANT if cfg.indicator == "constant" else INDICATOR_HENNEMANN,
            alpha_const=cfg.alphaconst)
        d = self.domain
        self.alpha = np.zeros(d.ne)
        self.fvm = subcell_interface_metrics(d) if self.shock.enabled else None
        self.t = 0.0
        self.steps = 0
        self.error = None
        self.kernel_seconds = {}
        self.comm_total = self.comm_covered = self.blocked_total = 0.0
        self.walltime = 0.0
        self.rhs_seconds = 0.0
        self.timing_active = False
        self.series_partials = []
        self.trace_rows = []
        self.mu0 = self.case_setup.mu0() if isinstance(self.case_setup, testcases.TGVSetup) \
            else gas.mu_ref
        d.U[...] = self.init_fn(d.x, gas)
        self._ready = False

    # -- device plumbing --------------------------------------------------
    def params(self):
        return self.domain.params(split=self.split, surf_solver=self.surf_solver_id,
                                  fv_solver=self.solver_id,
                                  shock=self.shock if self.shock.enabled else None,
                                  source=self.source, exact=self.exact,
                                  cfl=self.cfg.cfl, cfl_visc=self.cfg.cflvisc)

    def _prepare(self):
        if self._ready:
            return
        dv = self.domain.device
        if self.fvm is not None:
            dv.set_fvm(self.fvm)
        self.prm = self.params()
        _lib.check(dv.lib.hdg_check_domain(dv.dptr, ctypes.byref(self.prm)), "hdg_check_domain")
        # LGL stages run element pass -> surface fluxes -> streaming update, except
        # Euler with shock capturing (one fused volume pass); mirrors api.cu stage_impl
        self.split_stage = dv.vol is not None and bool(self.prm.viscous or not self.prm.shock)
        if self.comm is None and self.domain.sides_mpi.size:
            raise ProtocolError("partition-boundary sides need a communicator (multi-rank run)")
        torch = dv.torch
        si = self.domain.sides_inner
        # every local side in order (closed single-rank meshes): no list indirection
        self.flux_sides = None if np.array_equal(si, np.arange(self.domain.ns)) \
            else dv.int_tensor(si)
        self.rk_work = torch.zeros_like(dv.U)
        self.time_dev = torch.zeros(2, dtype=torch.float64, device=dv.dev)
        self._ready = True

    # -- the time derivative ----------------------------------------------
    def rhs_device(self, U, Ut, t):
        """Ut = RHS(U) on the device (device tensors, stream-ordered, no sync)."""
        self._prepare()
        d, dv = self.domain, self.domain.device
        if self.comm is not None:
            return self.comm.rhs(self, U, Ut, t)
        if d.basis.node_type == "LGL":
            _lib.check(dv.lib.hdg_rhs(dv.dptr, ctypes.byref(self.prm), _lib.ptr(U), _lib.ptr(Ut), t,
                                      _lib.ptr(self.flux_sides), int(d.sides_inner.size),
                                      dv.sptr()), "hdg_rhs")
        else:
            self._rhs_gl(U, Ut, t)
        return Ut

    def _rhs_gl(self, U, Ut, t):
        """GL (standard form) path: explicit prolong, then the phase kernels."""
        d, dv = self.domain, self.domain.device
        lib, s = dv.lib, dv.sptr()
        _lib.check(lib.hdg_prolong(dv.dptr, _lib.ptr(U), _lib.ptr(dv.rows_inner),
                                   int(d.rows_inner.shape[0]), s), "hdg_prolong")
        if self.prm.viscous:
            _lib.check(lib.hdg_phase_lift(dv.dptr, ctypes.byref(self.prm), _lib.ptr(U), s),
                       "hdg_phase_lift")
        _lib.check(lib.hdg_fill_flux_traces(dv.dptr, ctypes.byref(self.prm),
                                            _lib.ptr(self.flux_sides), int(d.sides_inner.size),
                                            self.prm.surf_solver, s), "hdg_fill_flux_traces")
        _lib.check(lib.hdg_phase_volume(dv.dptr, ctypes.byref(self.prm), _lib.ptr(U), _lib.ptr(Ut),
                                        None, t, 0.0, 0.0, 0.0, _lib.MODE_STORE_UT, s),
                   "hdg_phase_volume")

    def stage_device(self, U, dU, i, first, next_dt=False):
        """One fused LSERK stage on the device (time/dt read from self.time_dev).
        next_dt: also fold the next step's local dt + isfinite of the updated U into
        dt_bits (the last stage of a step)."""
        d, dv = self.domain, self.domain.device
        sc = self.scheme
        flags = int(bool(first)) | (_lib.STAGE_NEXT_DT if next_dt else 0)
        if self.comm is not None:
            return self.comm.stage(self, U, dU, i, flags)
        if d.basis.node_type != "LGL":
            # GL: rhs into the scratch buffer, then the fused update kernel
            Ut = self._scratch()
            self._rhs_gl_time(U, Ut, i)
            _lib.check(dv.lib.hdg_lserk_update(_lib.ptr(U), _lib.ptr(dU), _lib.ptr(Ut), U.numel(),
                                               float(sc.A[i]), float(sc.B[i]), self._dt_host,
                                               int(first), dv.sptr()), "hdg_lserk_update")
            return
        _lib.check(dv.lib.hdg_stage(dv.dptr, ctypes.byref(self.prm), _lib.ptr(U), _lib.ptr(dU),
                                    _lib.ptr(self.time_dev), float(sc.A[i]), float(sc.B[i]),
                                    float(sc.c[i]), flags, _lib.ptr(self.flux_sides),
                                    int(d.sides_inner.size), dv.sptr()), "hdg_stage")

    def stage_phases(self, U, dU, i, first, hook=None, next_dt=False):
        """The same stage as :meth:`stage_device`, launched phase by phase so a
        caller can record events between the kernels (``hook(name)`` is called
        before each phase and once at the end with ``None``)."""
        d, dv = self.domain, self.domain.device
        sc, lib, s = self.scheme, dv.lib, dv.sptr()
        prm = ctypes.byref(self.prm)
        visc = self.split_stage
        if visc:
            hook and hook("elem")
            _lib.check(lib.hdg_phase_elem(dv.dptr, prm, _lib.ptr(U), s), "hdg_phase_elem")
        hook and hook("flux")
        _lib.check(lib.hdg_phase_flux(dv.dptr, prm, _lib.ptr(U), _lib.ptr(self.flux_sides),
                                      int(d.sides_inner.size), self.prm.surf_solver, s),
                   "hdg_phase_flux")
        hook and hook("update" if visc else "volume")
        mode = _lib.MODE_LSERK_FIRST if first else _lib.MODE_LSERK
        if next_dt:
            mode |= 64 << 4     # the next step's local dt in the update epilogue
        fn = lib.hdg_phase_update if visc else lib.hdg_phase_volume
        _lib.check(fn(dv.dptr, prm, _lib.ptr(U), _lib.ptr(dU), _lib.ptr(self.time_dev), 0.0,
                      float(sc.A[i]), float(sc.B[i]), float(sc.c[i]), mode, s), "stage phase")
        hook and hook(None)

    def _scratch(self):
        if getattr(self, "_ut_scratch", None) is None:
            self._ut_scratch = self.domain.device.torch.empty_like(self.domain.device.U)
        return self._ut_scratch

    def _rhs_gl_time(self, U, Ut, i):
        self._rhs_gl(U, Ut, self.t + self.scheme.c[i] * self._dt_host)

    def evaluate_rhs(self, t: float) -> np.ndarray:
        """RankWorker.evaluate_rhs (src/parallel.py:539-563): host d.U in, host d.Ut out."""
        t0 = time.perf_counter()
        self._prepare()
        d, dv = self.domain, self.domain.device
        dv.upload_state()
        if d.viscous:
            dv.ensure_gradients()
        dv.status.copy_(dv.status_init)
        Ut = self._scratch()
        self.rhs_device(dv.U, Ut, t)
        st = dv.status.cpu().numpy()
        self._raise_status(st)
        d.Ut[...] = Ut.cpu().numpy()
        if d.viscous:
            dv.download_gradients()
        if self.shock.enabled:
            self.alpha[:] = dv.alpha[:d.ne].cpu().numpy()
        if self.timing_active:
            self.rhs_seconds += time.perf_counter() - t0
        return d.Ut

    def _raise_status(self, st):
        d = self.domain
        if st[_lib.STATUS_BAD_PRIM]:
            d._raise_prim(st)
        if st[_lib.STATUS_PEER_TIMEOUT]:
            raise ProtocolError(f"rank {self.rank}: peer-memory exchange timed out")
        if st[_lib.STATUS_BAD_SIDE] >= 0:
            raise AdmissibilityError(
                f"rank {self.rank}: inadmissible trace state on local side {int(st[1])}")

    # -- time loop ----------------------------------------------------------
    def _compute_dt_device(self):
        """dt + non-finite check on the device (src/parallel.py:595-604), no host sync."""
        d, dv = self.domain, self.domain.device
        dv.dt_bits.fill_(0x7FF0000000000000)
        _lib.check(dv.lib.hdg_local_dt(dv.dptr, ctypes.byref(self.prm), _lib.ptr(dv.U),
                                       self.cfg.cfl, self.cfg.cflvisc, dv.sptr()), "hdg_local_dt")
        if self.comm is not None:
            self.comm.allreduce_dt(self)
        _lib.check(dv.lib.hdg_dt_finalize(dv.dptr, _lib.ptr(self.time_dev), self.cfg.tend,
                                          dv.sptr()), "hdg_dt_finalize")

    def step_device(self):
        """One full RK step, device resident (dt, stages, t += dt).

        The step's dt was reduced into dt_bits by the previous step's last stage
        (the folded _compute_dt of the updated U); the first step after U changed
        on the host runs the standalone dt pass. dt_finalize reads it, clips it to
        tend and resets the accumulator, so a step needs no dt kernel and no fill.
        """
        d, dv = self.domain, self.domain.device
        if not dv.dt_valid:
            dv.dt_bits.fill_(0x7FF0000000000000)
            _lib.check(dv.lib.hdg_local_dt(dv.dptr, ctypes.byref(self.prm), _lib.ptr(dv.U),
                                           self.cfg.cfl, self.cfg.cflvisc, dv.sptr()),
                       "hdg_local_dt")
            if self.comm is not None:
                self.comm.allreduce_dt(self)
        _lib.check(dv.lib.hdg_dt_finalize(dv.dptr, _lib.ptr(self.time_dev), self.cfg.tend,
                                          dv.sptr()), "hdg_dt_finalize")
        S = self.scheme.stages
        for i in range(S):
            self.stage_device(dv.U, self.rk_work, i, i == 0, next_dt=(i == S - 1))
        if self.comm is not None:
            self.comm.allreduce_dt(self)
        dv.dt_valid = True
        _lib.check(dv.lib.hdg_time_advance(_lib.ptr(self.time_dev), dv.sptr()),
                   "hdg_time_advance")

    def analyze(self, on_analyze=None):
        """RankWorker.analyze (src/parallel.py:606-629) on the device state.

        Viscous: one RHS evaluation refreshes the lifted gradients (as the
        reference); the element rows come from the device analysis kernel and
        are reduced on rank 0 in global element order. Outside the timed region.
        """
        d, dv = self.domain, self.domain.device
        g = None
        drop = False
        if d.viscous:
            drop = dv.g is None
            dv.ensure_gradients()
            self.rhs_device(dv.U, self._scratch(), self.t)
            g = dv.g
            if self.comm is None:   # multi-rank: surfaces at the next step's collective check
                self._raise_status(dv.status.cpu().numpy())
        parts = testcases.analysis_partials_device(d, dv.U, g, self.mu0)
        amax = 0.0
        if d.ne:
            a = dv.alpha[:d.ne].max().item() if self.shock.enabled else 0.0
            amax = float(a)
        if drop:
            dv.drop_gradients()   # production stages run without the debug outputs
        if self.comm is not None:
            rows = self.comm.gather_rows(parts)
            amax = self.comm.max_over_ranks(amax)
        else:
            rows = parts.cpu().numpy()
        U = alpha = None
        if on_analyze is not None:
            # the reference's gathered rows: U as (ne, n1^3 * 5), alpha as (ne, 1)
            # (src/parallel.py:621-623; its CLI reads alpha_rows[:, 0])
            Ur, ar = dv.U.reshape(d.ne, -1), dv.alpha[:d.ne].reshape(d.ne, 1)
            if self.comm is not None:
                U, alpha = self.comm.gather_rows(Ur), self.comm.gather_rows(ar)
            else:
                U, alpha = Ur.cpu().numpy(), ar.cpu().numpy()
        if self.rank == 0:
            setup = self.case_setup if isinstance(self.case_setup, testcases.TGVSetup) \
                else testcases.TGVSetup(mach=1.0, reynolds=1.0)
            q = testcases.reduce_tgv_quantities(rows, setup)
            q["t"] = self.t
            q["dt"] = getattr(self, "last_dt", 0.0)
            q["max_alpha"] = amax
            self.series_partials.append(q)
            if on_analyze is not None:
                on_analyze(self.t, q, U, alpha)

    def run(self, on_analyze=None):
        """Time loop (src/parallel.py:631-667) with device-resident state."""
        try:
            cfg = self.cfg
            self._prepare()
            d, dv = self.domain, self.domain.device
            torch = dv.torch
            self.evaluate_rhs(self.t)           # warm-up, as the reference
            dv.upload_state()
            dv.drop_gradients()                 # stages run without the API debug outputs
            self.time_dev[0] = self.t
            if not getattr(self, "resumed", False):
                # a resumed run's first row would repeat the interrupted run's last one
                # (same t; max_alpha from a warm-up RHS instead of the last RK stage)
                self.analyze(on_analyze)        # walltime excludes analysis (:638-640)
            dv.status.copy_(dv.status_init)
            tracer = None
            if self.comm is not None:
                from .exchange import StreamTracer
                tracer = self.comm.tracer = StreamTracer(torch, self.rank)
            lgl = d.basis.node_type == "LGL"
            pending_nonfinite = False
            while True:
                if cfg.maxsteps and self.steps >= cfg.maxsteps:
                    break
                if self.t >= cfg.tend - 1e-12:
                    break
                if pending_nonfinite:
                    # the folded dt pass of the last step saw a non-finite U: this is the
                    # reference's _compute_dt failure at the start of this step
                    raise NumericalFailure(
                        f"non-finite solution at t = {self.t:.6g}, step {self.steps}")
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                self.timing_active = True
                if not lgl:
                    self._compute_dt_device()
                    self._dt_host = float(self.time_dev[1].item())
                    for i in range(self.scheme.stages):
                        self.stage_device(dv.U, self.rk_work, i, i == 0)
                    _lib.check(dv.lib.hdg_time_advance(_lib.ptr(self.time_dev), dv.sptr()),
                               "hdg_time_advance")
                else:
                    self.step_device()
                tv = self.time_dev.cpu().numpy()
                # multi-rank: a stage kernel's error flag is agreed over the ranks
                # before anyone raises (every rank stops at the same step)
                st = dv.status.cpu().numpy() if self.comm is None \
                    else self.comm.agree_status(dv.status)
                self.timing_active = False
                self.walltime += time.perf_counter() - t0
                if tracer is not None:
                    tracer.collect()
                if not lgl and st[_lib.STATUS_NONFINITE]:
                    raise NumericalFailure(
                        f"non-finite solution at t = {self.t:.6g}, step {self.steps}")
                self._raise_status(st)
                self.last_dt = float(tv[1])
                self.steps += 1
                self.t = float(tv[0])
                pending_nonfinite = lgl and bool(st[_lib.STATUS_NONFINITE])
                if cfg.analyzeinterval and self.steps % cfg.analyzeinterval == 0:
                    self.analyze(on_analyze)
            if not cfg.analyzeinterval or self.steps % cfg.analyzeinterval != 0:
                self.analyze(on_analyze)
            d.U[...] = dv.U.cpu().numpy()
            if self.shock.enabled:
                self.alpha[:] = dv.alpha[:d.ne].cpu().numpy()
            if tracer is not None:
                self.comm_total, self.comm_covered = tracer.window_total, tracer.covered
                self.trace_rows = tracer.rows
                for k, v in tracer.kernel_seconds.items():
                    self.kernel_seconds[k] = self.kernel_seconds.get(k, 0.0) + v
                self.comm.tracer = None
        except BaseException as exc:   # noqa: BLE001 - surfaced by run_distributed
            self.error = exc


class Stepper:
    """Graph-captured RK step for the production / benchmark loop.

    Captures [dt reduction + finalize, all stages, t += dt] once; replaying it
    costs one graph launch per step and no host synchronisation.
    """

    def __init__(self, worker: RankWorker, use_graph: bool = True):
        self.w = worker
        worker._prepare()
        dv = worker.domain.device
        self.torch = dv.torch
        self.graph = None
        if use_graph and worker.domain.basis.node_type == "LGL" and worker.comm is None:
            s = self.torch.cuda.Stream()
            s.wait_stream(self.torch.cuda.current_stream())
            with self.torch.cuda.stream(s):
                worker.step_device()              # warm (sets smem attributes)
            self.torch.cuda.current_stream().wait_stream(s)
            self.torch.cuda.synchronize()
            g = self.torch.cuda.CUDAGraph()
            with self.torch.cuda.graph(g):
                worker.step_device()
            self.graph = g

    def step(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            self.w.step_device()


def _build_mesh(cfg: RunConfig) -> Mesh:
    if cfg.meshfile:
        return load_mesh_cache(cfg.meshfile)
    mesh = generate_box_mesh(cfg.meshx, cfg.meshy, cfg.meshz,
                             [(cfg.x0, cfg.x1), (cfg.y0, cfg.y1), (cfg.z0, cfg.z1)],
                             (cfg.periodicx, cfg.periodicy, cfg.periodicz))
    if cfg.curveamplitude:
        mesh = curve_mesh(mesh, cfg.curveamplitude)
    return mesh


def restore_snapshot(worker: RankWorker, path: str) -> float:
    """Resume from an HDGF snapshot (io.write_snapshot of a run's U, t, alpha).

    The reference has no restart; the file is its own HDGF format
    (src/io.py:24-55). Each rank takes its SFC element range of the global field
    (mmap, so only its rows are read) and the snapshot time; the continued run is
    bitwise the uninterrupted one (tests/test_gpu_analysis.py). The blending
    factors are informational: alpha is recomputed from U every stage.
    """
    from .io import SnapshotError, read_snapshot
    d = worker.domain
    U, t, alpha = read_snapshot(path, mmap=True)
    n1 = d.basis.N + 1
    nvar = d.U.shape[-1]
    if U.shape[1:] != (n1, n1, n1, nvar):
        raise SnapshotError(f"snapshot field {U.shape[1:]} does not match N = {n1 - 1}, "
                            f"{nvar} variables")
    lo, hi = d.lo, d.hi
    if U.shape[0] != worker.n_elem_global:
        raise SnapshotError(f"snapshot has {U.shape[0]} elements, the mesh "
                            f"{worker.n_elem_global}")
    d.U[...] = U[lo:hi]
    if worker.shock.enabled:
        worker.alpha[:] = alpha[lo:hi]
    worker.t = float(t)
    worker.resumed = True
    return worker.t


def run_distributed(cfg: RunConfig, mesh: Mesh = None, on_analyze=None) -> RunResult:
    """Run the configured case (src/parallel.py:680-744).

    Single process: nranks must be 1 (one GPU). Under torchrun (torch.distributed
    initialised with world size == cfg.nranks) each process runs its rank and
    rank 0 returns the gathered result.
    """
    cfg.validate()
    basis = build_basis(cfg.n, cfg.nodetype)
    gas = cfg.gas()
    if mesh is None:
        mesh = _build_mesh(cfg)
    if mesh.J is None or mesh.basis is not basis:
        compute_metrics(mesh, basis)
    n_ranks = cfg.nranks
    if n_ranks > mesh.nelem:
        raise ValueError(f"{n_ranks} ranks exceed {mesh.nelem} elements")
    parts = partition_sfc(mesh, n_ranks)
    elem_rank = np.empty(mesh.nelem, dtype=np.int64)
    for p in parts:
        elem_rank[p.lo:p.hi] = p.rank
    transport = Transport(n_ranks)
    case = testcases.build_case(cfg)
    comm, rank = None, 0
    if n_ranks > 1:
        from .exchange import make_exchange
        comm = make_exchange(n_ranks)
        rank = comm.rank
    w = RankWorker(rank, mesh, basis, gas, parts[rank], elem_rank, cfg, transport,
                   SlotLimiter(1), case, comm=comm)
    if cfg.restartfile:
        restore_snapshot(w, cfg.restartfile)
    if comm is not None:
        comm.attach(w)
    w.run(on_analyze)
    err = w.error
    if comm is not None:
        err = comm.agree_error(err)
    if err is not None:
        cause = err
        while cause is not None:
            if isinstance(cause, (NumericalFailure, AdmissibilityError)):
                raise NumericalFailure(str(err)) from err
            cause = cause.__cause__
        raise err
    res = RunResult(t=w.t, steps=w.steps, series=w.series_partials, walltime=w.walltime,
                    n_ranks=n_ranks, n_dof=mesh.nelem * (cfg.n + 1) ** 3,
                    rk_stages=w.steps * w.scheme.stages, kernel_seconds=[w.kernel_seconds],
                    rhs_seconds=[w.rhs_seconds], message_counts=transport.messages_sent.copy(),
                    bytes_sent=transport.bytes_sent.copy(),
                    phase_counts=dict(transport.phase_counts),
                    phase_bytes=dict(transport.phase_bytes),
                    comm_stats=[{"window": w.comm_total, "covered": w.comm_covered,
                                 "blocked": w.blocked_total}],
                    trace=list(w.trace_rows))
    if comm is not None:
        res.U, res.alpha, res.walltime = comm.gather_result(w)
        stats = comm.gather_objects(({"window": w.comm_total, "covered": w.comm_covered,
                                      "blocked": w.blocked_total}, w.kernel_seconds,
                                     [tuple(vars(r).values()) for r in w.trace_rows]))
        res.comm_stats = [a for a, _, _ in stats]
        res.kernel_seconds = [b for _, b, _ in stats]
        from .exchange import TraceRow
        res.trace = [TraceRow(*row) for _, _, rows in stats for row in rows]
    else:
        res.U = w.domain.U.copy()
        res.alpha = w.alpha.copy()
    if comm is not None:
        comm.close()
    return res
