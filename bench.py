"""Benchmark: FP64 DGSEM RK steps on B200 (BASELINE.json metric: PID and DOF-updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

One "step" = one full low-storage RK step of the time loop (dt reduction +
all RK stages, each stage = element pass (prims, BR1 lifting, split volume
integral) + surface fluxes + streaming surface-integral/Jacobian/LSERK update),
on synthetic TGV input of the named configuration, random-free and fully
device resident. Under torchrun (N > 1) each rank owns
an SFC partition and face data moves every stage through the NVLink peer-memory
exchange (NCCL point-to-point fallback; paper_2404_12703_b200/exchange.py); times
are CUDA events, max over ranks.

Prints ONE JSON line (rank 0). ``--impl reference`` times the reference's CPU
algorithm (the bit-exact C oracle port, oracle/) on the host cores instead.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TWO_PI = 2.0 * np.pi

# name -> (description, RunConfig kwargs, mesh (nx,ny,nz) at 1 GPU, curved+flipped)
CONFIGS = {
    "c1": ("Euler MMS convergence case, N=3, 4^3 periodic, GL standard form, CK(5,4)",
           dict(testcase="mms", n=3, nodetype="GL", operator="standard", x0=-1.0, x1=1.0,
                y0=-1.0, y1=1.0, z0=-1.0, z1=1.0), (4, 4, 4), False),
    "c2": ("TGV Ma=0.1 Re=1600 Navier-Stokes, N=7, 32^3 elements, split form (KEP) + LLF-split, "
           "BR1, CK(5,4)",
           dict(testcase="tgv", n=7, mach=0.1, reynolds=1600.0, muref=1.0 / 1600.0),
           (32, 32, 32), False),
    "c3": ("TGV Ma=1.25 NS Sutherland, N=5, 64^3, FV-subcell shock capturing (Hennemann)",
           dict(testcase="tgv", n=5, mach=1.25, muref=1.0 / 1600.0, viscosity="sutherland",
                tref=1.0 / (1.4 * 1.25 ** 2 * 287.058), shockcapture=True),
           (64, 64, 64), False),
    "c3fv": ("TGV Ma=1.25 NS Sutherland, N=5, 64^3, FV subcell on every element (alpha=0.3)",
             dict(testcase="tgv", n=5, mach=1.25, muref=1.0 / 1600.0, viscosity="sutherland",
                  tref=1.0 / (1.4 * 1.25 ** 2 * 287.058), shockcapture=True,
                  indicator="constant", alphaconst=0.3), (64, 64, 64), False),
    "c4": ("curved randomly flipped hex mesh (all orientation codes), NS N=4, 1.0M DOF/GPU",
           dict(testcase="tgv", n=4, mach=0.1, muref=1.0 / 1600.0), (20, 20, 20), True),
    "c5": ("TGV N=7 strong-scaling mesh, 70^3 elements (175.6M DOF)",
           dict(testcase="tgv", n=7, mach=0.1, muref=1.0 / 1600.0), (70, 70, 70), False),
    "euler7": ("TGV Ma=0.1 Euler, N=7, 32^3, split form", dict(testcase="tgv", n=7, mach=0.1),
               (32, 32, 32), False),
}

# algorithmic HBM bytes per DOF of each kernel launch (FP64, this design)
def kernel_bytes(N, viscous, split=True):
    face = 1.0 / (N + 1)       # face nodes per DOF, per element face
    if not viscous and split:
        # Euler A: U, Ja, 1/J -> Vol; B: both traces, nvec+ssurf -> f*; C as NS
        return {"elem": 40 + 72 + 8 + 40, "flux": 3 * face * (80 + 32 + 40),
                "update": 40 + 6 * face * 40 + 8 + 40 + 40 + 40 + 40,
                "dt_per_step": 40 + 72 + 8}
    if viscous:
        # A: U, Ja, 1/J, neighbour traces + nvec/ssurf on 6 faces -> Vol + face viscous fluxes
        elem = 40 + 72 + 8 + 6 * face * (40 + 32) + 40 + 6 * face * 32
        # B: both traces, nvec+ssurf, both face viscous fluxes -> f*
        flux = 3 * face * (80 + 32 + 64 + 40)
        # C: Vol, f* on 6 faces, 1/J, dU, U -> dU, U; the last stage of a step also
        # reads Ja + J for the folded next-step dt (80 B/DOF, 1 launch in n_stages)
        update = 40 + 6 * face * 40 + 8 + 40 + 40 + 40 + 40
        return {"elem": elem, "flux": flux, "update": update, "dt_fold_per_step": 72 + 8}
    vol = 40 + 72 + 8 + 40 + 40 + 40 + 6 * 40 * face
    flux = 3 * face * (80 + 32 + 40)
    return {"volume": vol, "flux": flux, "dt_per_step": 40 + 72 + 8}


def survey_bytes(N, viscous):
    """SURVEY §8(d) ideal-fusion algorithmic bytes per DOF per RK stage."""
    n1 = N + 1
    return 360 + 2664 / n1 if viscous else 240 + 696 / n1


def mesh_counts(base, n_gpus, weak):
    nx, ny, nz = base
    if not weak:
        return base
    # C4 weak scaling: double x, then y, then z (1/2/4/8 GPUs)
    k = int(round(np.log2(n_gpus)))
    for i in range(k):
        if i % 3 == 0:
            nx *= 2
        elif i % 3 == 1:
            ny *= 2
        else:
            nz *= 2
    return (nx, ny, nz)


def gpu_local_cpus(dev):
    """CPUs on the GPU's NUMA node (sysfs local_cpulist of its PCI function), or None."""
    try:
        import torch
        p = torch.cuda.get_device_properties(dev)
        path = (f"/sys/bus/pci/devices/{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:"
                f"{p.pci_device_id:02x}.0/local_cpulist")
        cpus = set()
        with open(path) as f:
            for part in f.read().strip().split(","):
                lo, _, hi = part.partition("-")
                cpus.update(range(int(lo), int(hi or lo) + 1))
        return cpus or None
    except (OSError, ValueError, AttributeError):
        return None


def pinned_near_gpu(shape, dev):
    """Pinned host buffer whose pages sit on the GPU's NUMA node: cudaHostAlloc faults the
    pages in from the calling thread, so the thread is moved to the GPU-local CPUs for the
    allocation (first touch) and restored afterwards. Returns (tensor, cpus used or None)."""
    import torch
    cpus = gpu_local_cpus(dev)
    old = os.sched_getaffinity(0)
    use = (cpus & old) if cpus else None
    try:
        if use:
            os.sched_setaffinity(0, use)
        t = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        t.zero_()
    finally:
        if use:
            os.sched_setaffinity(0, old)
    return t, use


def build_config(name, n_gpus):
    from paper_2404_12703_b200.config import RunConfig
    desc, kw, base, curved = CONFIGS[name]
    weak = name == "c4"
    nx, ny, nz = mesh_counts(base, n_gpus, weak)
    kw = dict(kw)
    if "x0" not in kw:
        kw.update(x0=0.0, x1=TWO_PI, y0=0.0, y1=TWO_PI, z0=0.0, z1=TWO_PI)
    cfg = RunConfig(meshx=nx, meshy=ny, meshz=nz, nranks=n_gpus, tend=1e9,
                    analyzeinterval=0, **kw)
    return desc, cfg, curved, weak


def build_mesh(cfg, curved):
    from paper_2404_12703_b200 import mesh as mm
    m = mm.generate_box_mesh(cfg.meshx, cfg.meshy, cfg.meshz,
                             [(cfg.x0, cfg.x1), (cfg.y0, cfg.y1), (cfg.z0, cfg.z1)], (True,) * 3)
    if curved:
        m = mm.curve_mesh(mm.random_flips(m, seed=0), 0.05)
    return m


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:   # sampling is live
                time.sleep(0.01)
            self.rows.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if not self.rows:
                # timed region shorter than the 50 ms period: one sample right after it
                try:
                    out = subprocess.run(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=10).stdout
                    self.rows = [[c.strip() for c in line.split(",")]
                                 for line in out.splitlines() if line.strip()]
                    self.post = True
                except (OSError, subprocess.TimeoutExpired):
                    pass

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        active = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower().startswith("active"):
                    active.add(n)
        pw = [float(r[2]) for r in self.rows if len(r) >= 3 and r[2].replace(".", "").isdigit()]
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(self.rows[0][1]),
               "reasons": sorted(active), "samples": len(sm),
               "power_w_median": float(np.median(pw)) if pw else None}
        if getattr(self, "post", False):
            out["sampled"] = "right after the timed region (shorter than one 50 ms period)"
        return out


def cpu_model():
    """Host CPU model name (/proc/cpuinfo) for the cpu_baseline line."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# geometry: the reference's own numpy curl-form metrics (bit-identical) up to C2 size; the
# cuBLAS / torch evaluation of the same formulas (~1e-15 relative) for the larger meshes
NUMPY_METRICS_MAX_NODES = 1 << 25


def metrics_backend(cfg, nelem):
    return "numpy" if nelem * (cfg.n + 1) ** 3 <= NUMPY_METRICS_MAX_NODES else "torch"


def oracle_domain_for(cfg, curved, mesh=None):
    """The bit-exact C oracle of the reference on the configuration's mesh and initial state
    (mesh: the benchmark's own mesh with its metrics, reused)."""
    import oracle
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.mesh import compute_metrics
    from paper_2404_12703_b200.operator import Domain
    from paper_2404_12703_b200.testcases import build_case
    basis = build_basis(cfg.n, cfg.nodetype)
    if mesh is None:
        m = build_mesh(cfg, curved)
        compute_metrics(m, basis, backend=metrics_backend(cfg, m.nelem))
    else:
        m = mesh
    gas = cfg.gas()
    d = Domain(m, basis, gas)
    init, bc, source, _ = build_case(cfg)
    od = oracle.OracleDomain(d, basis, gas)
    od.U[...] = init(d.x, gas)
    split = cfg.operator == "split"
    solver = 1 if cfg.riemann == "hllc" else 0
    kw = dict(split=split, surf_solver=2 if (split and solver == 0) else solver, solver=solver,
              shock=(dict(constant=cfg.indicator == "constant", alpha_const=cfg.alphaconst,
                          alpha_max=cfg.alphamax, alpha_min=cfg.alphamin)
                     if cfg.shockcapture else None), source=source)
    return m, od, kw


def parity_vs_oracle(od, kw, Ut_gpu, Ut_exact=None):
    """One full-size RHS of the benchmark's production path vs the oracle on the same
    initial state (SURVEY §8d parity protocol: normwise and per-variable inf-norms), and
    the exact kernel set's RHS of the same state checked bit for bit."""
    t0 = time.perf_counter()
    U0 = od.U.copy()
    ref = od.evaluate_rhs(0.0, **kw).copy()
    od.U[...] = U0
    a, b = Ut_gpu.reshape(-1, 5), ref.reshape(-1, 5)
    per_var = np.max(np.abs(a - b), axis=0) / np.maximum(np.max(np.abs(b), axis=0), 1e-300)
    out = {"normwise": float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-300)),
           "per_variable": [float(x) for x in per_var],
           "tolerance": "1e-12, or 2x the reference's own error vs an extended-precision "
                        "evaluation where the RHS is ill conditioned (Ma 0.1: the unperturbed "
                        "vortex's Ut is ~1e-4 of its pressure terms; tests/test_gpu_parity.py)",
           "what": "||Ut_fast - Ut_oracle||_inf / ||Ut_oracle||_inf, one RHS of the full "
                   "benchmark mesh at its initial state, production (fast, FMA) kernel set",
           "oracle_seconds": time.perf_counter() - t0}
    if Ut_exact is not None:
        out["exact_set_bitwise"] = bool(np.array_equal(Ut_exact, ref))
        out["exact_set_normwise"] = float(np.max(np.abs(Ut_exact - ref)) /
                                          max(float(np.max(np.abs(ref))), 1e-300))
    return out


def cpu_reference(cfg, curved, steps, warmup, threads=None, per_stage=False, prepared=None):
    """The reference's CPU algorithm (bit-exact C oracle, OpenMP) on the host cores.

    One sample = one full RK step (dt + all stages) of the same configuration.
    Returns (DOF-updates/s, seconds per step list, cores)."""
    import oracle
    from paper_2404_12703_b200.timedisc import get_scheme
    cores = threads or os.cpu_count()
    os.environ["OMP_NUM_THREADS"] = str(cores)
    m, od, kw = prepared or oracle_domain_for(cfg, curved)
    sc = get_scheme(cfg.rkscheme)
    times = []
    t = 0.0
    if per_stage:
        # one sample = one RK stage (RHS + the reference's numpy-order LSERK update)
        import ctypes
        work = np.zeros_like(od.U)
        lib = oracle.lib()
        dt = 1e-4
        for k in range(warmup + steps):
            i = k % sc.stages
            t0 = time.perf_counter()
            Ut = od.evaluate_rhs(t + sc.c[i] * dt, **kw)
            lib.orc_lserk(od.U.ctypes.data_as(ctypes.c_void_p), work.ctypes.data_as(ctypes.c_void_p),
                          Ut.ctypes.data_as(ctypes.c_void_p), od.U.size, float(sc.A[i]),
                          float(sc.B[i]), dt, int(i == 0))
            if k >= warmup:
                times.append(time.perf_counter() - t0)
        dof = m.nelem * (cfg.n + 1) ** 3
        return dof / float(np.mean(times)), times, cores, dof
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        t, _ = od.rk_steps(1, sc, cfg.cfl, cfg.cflvisc, t=t, **kw)
        if k >= warmup:
            times.append(time.perf_counter() - t0)
    dof = m.nelem * (cfg.n + 1) ** 3
    return dof * sc.stages / float(np.mean(times)), times, cores, dof


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--exact", action="store_true", help="bit-exact (-fmad=false) kernel set")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    # exactly one JSON line on stdout: route everything else (NCCL's C-level version
    # banner, library prints) to stderr until the result is printed
    sys.stdout.flush()
    real_stdout = os.dup(1)
    os.dup2(2, 1)

    def emit(obj):
        sys.stdout.flush()
        os.dup2(real_stdout, 1)
        print(json.dumps(obj), flush=True)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    desc, cfg, curved, weak = build_config(args.config, args.gpus)

    if args.impl == "reference":
        if rank != 0:
            return
        value, times, cores, dof = cpu_reference(cfg, curved, args.steps, args.warmup,
                                                 per_stage=True)
        out = {
            "metric": "DOF-updates/s", "value": value, "unit": "DOF*stage/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (TGV initial field)",
            "pid_s": 1.0 / value,
            "config": {"workload": args.config, "description": desc, "dof": dof,
                       "elements": cfg.meshx * cfg.meshy * cfg.meshz, "N": cfg.n,
                       "step": "one RK stage (RHS + LSERK update) of the full mesh per sample",
                       "dt_pass": "excluded: the per-step dt reduction (one extra pass over U, "
                                  "~1/5 of an RHS) is not in the CPU samples, while the GPU "
                                  "arm's steps include it (conservative for the GPU ratio)"},
            "cpu_baseline": {"value": value, "unit": "DOF*stage/s", "cores": cores,
                             "kind": "port", "cpu_model": cpu_model(),
                             "sample": f"{args.steps} RK stages (RHS + LSERK update) of the full "
                                       f"{args.config} mesh ({dof} DOF): bit-exact C oracle of "
                                       "the reference's numba kernels, OpenMP on all host cores"},
            "e2e": {"value": value, "unit": "DOF*stage/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        emit(out)
        return

    import torch
    torch.cuda.set_device(local_rank)
    from paper_2404_12703_b200 import _lib
    from paper_2404_12703_b200 import testcases
    from paper_2404_12703_b200.basis import build_basis
    from paper_2404_12703_b200.mesh import compute_metrics, partition_sfc
    from paper_2404_12703_b200.parallel import RankWorker, SlotLimiter, Transport

    comm = None
    if world > 1:
        from paper_2404_12703_b200.exchange import make_exchange
        comm = make_exchange(world)

    t_setup = time.perf_counter()
    m = build_mesh(cfg, curved)
    basis = build_basis(cfg.n, cfg.nodetype)
    geometry = metrics_backend(cfg, m.nelem)
    compute_metrics(m, basis, backend=geometry)
    parts = partition_sfc(m, world)
    elem_rank = np.repeat(np.arange(world), [p.n_elems for p in parts])
    w = RankWorker(rank, m, basis, cfg.gas(), parts[rank], elem_rank, cfg, Transport(world),
                   SlotLimiter(1), testcases.build_case(cfg), comm=comm, exact=args.exact)
    if comm is not None:
        comm.attach(w)
    w._prepare()
    d, dv = w.domain, w.domain.device
    dv.upload_state()
    w.time_dev.zero_()
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()
    n_stages = w.scheme.stages
    dof_total = m.nelem * (cfg.n + 1) ** 3
    dof_local = d.ne * (cfg.n + 1) ** 3

    ev_pool = []

    def hook_factory(store):
        state = {"name": None, "ev": None}

        def hook(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            if state["name"] is not None:
                store.append((state["name"], state["ev"], e))
            state["name"], state["ev"] = name, e
        return hook

    def step(store=None):
        # RankWorker.step_device: dt_finalize of the dt the previous step's last stage
        # folded into its update epilogue, the stages, t += dt (the phase-by-phase
        # variant below records events between the kernels for the per-kernel table)
        if store is None or comm is not None:
            w.step_device()
            return
        if not dv.dt_valid:
            w.step_device()
            return
        _lib.check(dv.lib.hdg_dt_finalize(dv.dptr, _lib.ptr(w.time_dev), cfg.tend, dv.sptr()),
                   "dt_finalize")
        for i in range(n_stages):
            w.stage_phases(dv.U, w.rk_work, i, i == 0, hook=hook_factory(store),
                           next_dt=(i == n_stages - 1))
        _lib.check(dv.lib.hdg_time_advance(_lib.ptr(w.time_dev), dv.sptr()), "time_advance")

    def barrier():
        if comm is not None:
            comm.barrier()
        torch.cuda.synchronize()

    # parity (rank 0 at N=1): the production path's RHS at the initial state, compared
    # with the oracle below (after the timed region)
    Ut0 = Ut0x = None
    if world == 1 and not args.no_cpu_baseline and not args.no_parity:
        Ut_dev = torch.empty_like(dv.U)
        w.rhs_device(dv.U, Ut_dev, 0.0)
        Ut0 = Ut_dev.cpu().numpy()
        # the same RHS through the exact (-fmad=false) kernel set: bitwise the oracle
        ex = w.prm.exact
        w.prm.exact = 1
        w.rhs_device(dv.U, Ut_dev, 0.0)
        w.prm.exact = ex
        Ut0x = Ut_dev.cpu().numpy()
        del Ut_dev
        dv.status.copy_(dv.status_init)

    for _ in range(args.warmup):
        step()
    barrier()
    # multi-GPU over peer memory: every kernel of a step (exchanges and the dt
    # all-reduce included) is ours, so the whole step replays as one CUDA graph
    graph = None
    from paper_2404_12703_b200.exchange import PeerExchange
    if isinstance(comm, PeerExchange) and os.environ.get("HEXDG_GRAPH", "1") != "0":
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        c0 = dv.lib.hdg_launch_count()
        with torch.cuda.graph(graph, stream=side):
            step()
        graph_launches = dv.lib.hdg_launch_count() - c0   # kernels per replayed step
        torch.cuda.synchronize()

        def step(store=None):
            graph.replay()
        step()
        barrier()
    phases = []
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        barrier()
        launches0 = dv.lib.hdg_launch_count()
        start.record(stream)
        for _ in range(args.steps):
            step(phases)
        end.record(stream)
        barrier()
        launches = dv.lib.hdg_launch_count() - launches0
        if graph is not None:
            launches = graph_launches * args.steps
    ms = start.elapsed_time(end)
    # the same steps through the exact (-fmad=false) kernel set, bit-identical to the
    # reference (1 GPU, default fast run only): its throughput next to the fast set's
    exact_set = None
    if world == 1 and not args.exact and graph is None:
        w.prm.exact = 1
        for _ in range(2):
            w.step_device()
        torch.cuda.synchronize()
        ex0 = torch.cuda.Event(enable_timing=True)
        ex1 = torch.cuda.Event(enable_timing=True)
        ex0.record(stream)
        for _ in range(args.steps):
            w.step_device()
        ex1.record(stream)
        torch.cuda.synchronize()
        w.prm.exact = 0
        ms_x = ex0.elapsed_time(ex1)
        exact_set = {"value": dof_total * n_stages * args.steps / (ms_x * 1e-3),
                     "unit": "DOF*stage/s", "ms_per_step": ms_x / args.steps,
                     "parity": "bit-identical to the reference (parity.exact_set_bitwise at "
                               "full size; tests/test_gpu_parity.py goldens)"}
    if comm is not None:
        ms = comm.max_over_ranks(ms)
    st = dv.status.cpu().numpy()
    if st[_lib.STATUS_PEER_TIMEOUT]:
        raise SystemExit("peer-memory exchange timed out during the benchmark")
    if st[_lib.STATUS_NONFINITE] or st[_lib.STATUS_BAD_PRIM]:
        raise SystemExit(f"numerical failure during the benchmark: status {st}")
    per_kernel = {}
    for name, a, b in phases:
        per_kernel.setdefault(name, []).append(a.elapsed_time(b))
    ms_step = ms / args.steps
    value = dof_total * n_stages * args.steps / (ms * 1e-3)
    pid = ms * 1e-3 * world / (n_stages * args.steps * dof_total)

    # roofline of the dominant kernel (device events on its launch stream)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    kb = kernel_bytes(cfg.n, d.viscous, w.split_stage)
    kstats = {k: {"mean_ms": float(np.mean(v)), "launches": len(v),
                  "share": float(np.sum(v)) / ms if comm is None else None}
              for k, v in per_kernel.items()}
    for k in kstats:
        kstats[k]["achieved_gbs"] = kb[k] * dof_local / (kstats[k]["mean_ms"] * 1e-3) / 1e9
    if per_kernel:
        dom = max(per_kernel, key=lambda k: np.sum(per_kernel[k]))
        ach = kstats[dom]["achieved_gbs"]
    else:
        # multi-rank: no per-kernel events (the exchange interleaves); whole-step figure
        dom = "step"
        kb["step"] = survey_bytes(cfg.n, d.viscous) * n_stages
        ach = kb["step"] * dof_local / (ms_step * 1e-3) / 1e9
    traffic = flops = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = prof.get(args.config, {}).get(dom)
        flops = prof.get("fp64_flop_per_dof", {}).get(args.config, {}).get(dom)
    except (OSError, ValueError):
        pass
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": traffic,
                "bytes_per_dof": kb[dom], "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"
                if peaks else "fallback 6650 GB/s",
                "kernels": kstats,
                "step_alg_bytes_per_dof_stage_survey": survey_bytes(cfg.n, d.viscous),
                "step_frac_of_hbm_roofline":
                    survey_bytes(cfg.n, d.viscous) * value / world / 1e9 / hbm}
    if flops and per_kernel:
        # the element pass is FP64-issue bound, not HBM bound: its compute roofline
        # (FP64 flop per DOF from the ncu instruction counts of one launch, DFMA = 2)
        peak_tf, peak_src = 148 * 64 * 2 * 1965e6 / 1e12, "computed: 148 SM x 64 FMA x 2 x 1965 MHz"
        try:
            fp = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
            peak_tf, peak_src = float(fp["dfma_tflops"]), "measured"
        except (OSError, ValueError, KeyError):
            pass
        ach_tf = flops * dof_local / (kstats[dom]["mean_ms"] * 1e-3) / 1e12
        roofline["fp64"] = {"flop_per_dof": flops, "achieved": ach_tf, "peak": peak_tf,
                            "unit": "TFLOP/s", "frac": ach_tf / peak_tf,
                            "peak_source": peak_src,
                            "peak_file": "profiles/fp64_peak.json (DFMA microbenchmark, B200)",
                            "source": "profiles/ncu_traffic.json (ncu sass op counts)"}

    # end to end: pinned host U -> device, one RK step, device -> host U, per step.
    # The copies are split into element chunks on two copy streams so the
    # device->host read of step k and the host->device write of step k+1 run
    # full duplex (chunk i of step k+1 goes up as soon as chunk i of step k came
    # down); the step itself still starts only once all of its input is resident.
    e2e = None
    if not args.no_e2e:
        host_U, local_cpus = pinned_near_gpu(dv.U.shape, dv.U.device)
        host_U.copy_(dv.U)
        nbytes = host_U.numel() * 8
        n_chunks = 16 if d.ne >= 16 else 1
        bounds = np.linspace(0, d.ne, n_chunks + 1).astype(int)
        dev_chunks = [dv.U[a:b] for a, b in zip(bounds[:-1], bounds[1:])]
        host_chunks = [host_U[a:b] for a, b in zip(bounds[:-1], bounds[1:])]
        up, down = torch.cuda.Stream(), torch.cuda.Stream()
        down_done = [None] * n_chunks
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        up.wait_stream(stream)
        down.wait_stream(stream)
        for _ in range(args.steps):
            up_done = []
            for i in range(n_chunks):
                if down_done[i] is not None:
                    up.wait_event(down_done[i])
                with torch.cuda.stream(up):
                    dev_chunks[i].copy_(host_chunks[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(up)
                up_done.append(ev)
            for ev in up_done:
                stream.wait_event(ev)
            step()
            done = torch.cuda.Event()
            done.record(stream)
            down.wait_event(done)
            for i in range(n_chunks):
                with torch.cuda.stream(down):
                    host_chunks[i].copy_(dev_chunks[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(down)
                down_done[i] = ev
        stream.wait_stream(down)
        e1.record(stream)
        barrier()
        ms_e2e = e0.elapsed_time(e1)
        if comm is not None:
            ms_e2e = comm.max_over_ranks(ms_e2e)
        e2e = {"value": dof_total * n_stages * args.steps / (ms_e2e * 1e-3),
               "unit": "DOF*stage/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "ms_per_step": ms_e2e / args.steps,
               "api": "RankWorker stage path via the C ABI, host U in/out every step "
                      f"({n_chunks} chunks, full-duplex copy streams)",
               "host_buffer": ("pinned, first-touched on the GPU's NUMA node "
                               f"({len(local_cpus)} local CPUs)") if local_cpus
               else "pinned (GPU NUMA node unknown)"}

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            prepared = oracle_domain_for(cfg, curved, mesh=m)
            if Ut0 is not None:
                parity = parity_vs_oracle(prepared[1], prepared[2], Ut0, Ut0x)
            cval, ctimes, cores, _ = cpu_reference(cfg, curved, 1, 0, prepared=prepared)
            cpu = {"value": cval, "unit": "DOF*stage/s", "cores": cores, "kind": "port",
                   "cpu_model": cpu_model(),
                   "sample": f"1 full RK step ({n_stages} stages + dt) of the {args.config} mesh "
                             f"({dof_total} DOF), bit-exact C oracle of the reference kernels",
                   "seconds": float(ctimes[0])}
        except Exception as exc:  # noqa: BLE001 - the GPU number stands on its own
            cpu = {"value": None, "error": repr(exc)[:200]}

    if comm is not None:
        comm.close()
    if rank != 0:
        return
    out = {
        "metric": "DOF-updates/s", "value": value, "unit": "DOF*stage/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak" if weak else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (TGV initial field)",
        "pid_s": pid,
        "config": {"workload": args.config, "description": desc, "dof": dof_total,
                   "elements": m.nelem, "N": cfg.n, "rk": cfg.rkscheme,
                   "stages_per_step": n_stages, "parallelism": f"dd{world}",
                   "kernel_set": "exact" if args.exact else "fast",
                   "l2": "inputs larger than L2 (working set >> 126 MB), no flush needed",
                   "geometry": ("curl-form metrics by the reference's numpy formulas (bit-identical)"
                                if geometry == "numpy" else
                                "curl-form metrics by the same formulas on the GPU (torch/cuBLAS, "
                                "~1e-15 relative to the reference's numpy; oracle and GPU share them)"),
                   "setup_s": setup_s},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
        "exact_set": exact_set,
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    emit(out)


if __name__ == "__main__":
    main()
