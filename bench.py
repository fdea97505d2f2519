#!/usr/bin/env python
"""Benchmark: space-angle DOF-updates/s per sawtooth cycle (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]

Workload (default ``c4``): BASELINE config 4 — 1 group, cubic ConvFEM PG,
512 x 512 cells, 2048 ordinates (angle grid 32 x 32 -> n_a = 16), seeded 32 x 32
block materials, the largest configuration that fits one B200 and the one the
metric's 1/2/4/8-GPU scaling is quoted on.  A step is one sawtooth cycle
(flux/source assembly + the full multigrid cycle) of that solve, continuing the
solve's own trajectory from psi = 0 (warm-up cycles first).  The per-cycle fields
(2.3 GB each) exceed the 126 MB L2, so no flush is needed between steps.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the CPU oracle port of
the reference (oracle/, NumPy fp64, the reference is pure Python) on a bounded
sample of the same workload.
"""

import argparse
import json
import os

# load every kernel image when the library is registered, not on its first launch: a
# kernel first used inside the timed region (the first frozen-cycle residual, say)
# would otherwise put its module load into that step's device time
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# The CPU legs (the reference arm and the cpu_baseline subprocess) run the reference's
# single-threaded NumPy code (R/cli.py:61-62 parses --threads and never uses it): pin
# every BLAS / OpenMP pool to one thread BEFORE numpy loads, so "1 core" is enforced.
CPU_THREAD_VARS = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS",
                   "NUMEXPR_NUM_THREADS", "VECLIB_MAXIMUM_THREADS")
if "--cpu-sample" in sys.argv or ("--impl" in sys.argv and "reference" in sys.argv):
    for _v in CPU_THREAD_VARS:
        os.environ[_v] = "1"

import numpy as np  # noqa: E402

HBM_FALLBACK_GBS = 6650.0


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured", d
    return HBM_FALLBACK_GBS, "fallback", {}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.first = 0

    def start(self):
        """Launch the sampler (before the warm-up: nvidia-smi takes longer to come up
        than a short timed region lasts) and wait for its first row."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        t0 = time.perf_counter()
        while not self.rows and time.perf_counter() - t0 < 10.0:
            time.sleep(0.01)

    def mark(self):
        """The timed region starts: only rows from here on count."""
        self.first = len(self.rows)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t0 = time.perf_counter()     # a region shorter than the period: its next row
        while len(self.rows) <= self.first and time.perf_counter() - t0 < 0.2:
            time.sleep(0.005)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.rows = self.rows[self.first:]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, n in enumerate(names):
                if r[4 + k].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ----------------------------------------------------------------------------- workload
def workload(name, nx=None, world=1, n_a=None, slabs=None):
    """BASELINE config by name; c5w is the weak-scaling C5 variant (512 x 512 cells per
    rank, stacked along x), c5 the full 1024 x 1024 C5 (strong scaling, >= 4 GPUs: one
    fp32 field is 60.8 GB)."""
    from paper_2301_09991_b200 import benchmarks as B
    if name == "c1":
        return B.c1()
    if name == "c2":
        return B.c2()
    if name == "c3":
        return B.c3()
    if name == "c4":
        kw = {"n_a": n_a} if n_a else {}
        return B.c4(**kw) if nx is None else B.c4(nx=nx, blocks=nx // 16, **kw)
    if name == "c5w":
        # slabs: build the weak problem of that many ranks whatever the world size (the
        # single-domain reference of a DD plumbing check); n_a: fewer ordinates (checks)
        return B.c5_weak(slabs or world, **({"n_a": n_a} if n_a else {}))
    if name == "c5":
        if world < 4 and not n_a:
            raise SystemExit("c5 (1024^2 x 2048 ordinates x 7 groups, 60.8 GB per fp32 "
                             "field) needs >= 4 GPUs; use c5w for the per-GPU weak variant")
        return B.c5(**({"n_a": n_a} if n_a else {}))     # n_a: plumbing checks only
    raise SystemExit(f"unknown config {name}")


def options_for(P, pd, dtype, cycles=None, fold=False):
    o = dict(pd.options)
    pg = o.pop("pg", None)
    if cycles is not None:
        o["mg_iters"] = cycles
    return P.SolverOptions(**o, pg=P.PGConfig(**(pg or {})), dtype=dtype, fold_z=fold)


def per_dof_bytes(kernel, esz, eng=None):
    """Algorithmic bytes per finest DOF of one launch: the fused sweep reads
    psi, delta, kx, ky and writes psi (20 B fp32) — or, with the correction folded into
    the iterate (CycleEngine.fold_delta: the finest smoother already formed psi' = psi -
    delta), reads psi', kx, ky and writes psi (16 B)."""
    sweep = getattr(eng, "sweep_elems", 5) if eng is not None else 5
    return {"pg_sweep": sweep, "pg_residual": 4, "pg_residual+ema": 6, "pg_diffusivity": 5,
            "ema": 3, "upwind_residual": 2}.get(kernel, 0) * esz


def fp32_peak_tflops(peaks):
    """CUDA-core FP32 peak, derived (the driver measures no FP32 figure): 148 SMs x 128
    FP32 lanes x 2 flops x the measured maximum SM clock."""
    return 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12


def sweep_roofline(pd, ldof, esz, eng, ms_k, peak, peak_kind, peaks):
    """Roofline of the fused PG sweep (K5) from its event-timed launch duration: HBM
    (algorithmic bytes / duration vs the measured copy bandwidth) and FP32 (the
    reference formulation's 32T + 22 flops per DOF, vs the derived FP32 peak).
    The bound is whichever roof is lower for this order: bytes/BW vs flops/P."""
    bpl = per_dof_bytes("pg_sweep", esz, eng) * ldof
    order = pd.options.get("order", 1)
    flops = (32 * (2 * order + 1) + 22) * ldof
    fpk = fp32_peak_tflops(peaks)
    t_hbm = bpl / (peak * 1e9)
    t_fp = flops / (fpk * 1e12)
    hbm = {"achieved": bpl / (ms_k * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
           "frac": t_hbm / (ms_k * 1e-3), "bytes_per_launch": bpl,
           "bytes_per_dof": bpl / ldof,
           "peak_source": ("measured (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured"
                           else "fallback 6.65 TB/s")}
    fp = {"achieved": flops / (ms_k * 1e-3) / 1e12, "peak": fpk, "unit": "TFLOP/s",
          "frac": t_fp / (ms_k * 1e-3), "flops_per_dof": flops / ldof,
          "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x sm_max_mhz (no measured FP32 peak)"}
    return hbm, fp, ("fp32" if t_fp > t_hbm else "hbm"), max(t_hbm, t_fp) / (ms_k * 1e-3)


def bytes_model(pd, hier, live):
    """Algorithmic fp32 bytes per cycle."""
    lv = [l.grid.nx * l.grid.ny * l.quad.n_dir * pd.n_groups for l in hier.levels]
    n0, coarse = lv[0], sum(lv[1:])
    if pd.options["scheme"] == "upwind" or pd.options.get("pg", {}).get("alpha_r", 3.0) == 0.0:
        return 28 * n0 + 16 * coarse
    # live: K2 20 + K3 16 + finest correction 8 + K5 20; frozen: the EMA (12 B standalone)
    # shares the residual's psi read (R/multigrid.py:282 then :287), 8 B -> 52
    return (64 if live else 52) * n0 + 16 * coarse


# ----------------------------------------------------------------------------- reference arm
def cpu_sample_problem(name, arm=False):
    """Bounded CPU sample of the workload for the reference (fp64 NumPy, 1 core).

    c4: the cpu_baseline leg runs one cycle of the 128 x 128, n_a = 8 instance of the
    C4 generator (~20 s on one core); the reference arm's steps use
    the 64 x 64, n_a = 8 instance (~2-3 s per cycle, so W + K steps stay within
    minutes).  Same generator, order, ordinates per face and material statistics."""
    from paper_2301_09991_b200 import benchmarks as B
    if name == "c4":
        if arm:
            return B.c4(nx=64, blocks=4, n_a=8, cycles=1), "c4 generator at 64x64 cells, n_a=8 (512 ordinates), cubic PG"
        return B.c4(nx=128, blocks=8, n_a=8, cycles=1), "c4 generator at 128x128 cells, n_a=8 (512 ordinates), cubic PG"
    if name == "c2":
        return B.c2(nx=64, blocks=8, n_a=8, cycles=1), "c2 generator at 64x64 cells, n_a=8, quadratic PG"
    if name == "c1":
        return B.c1(cycles=1), "c1 full size"
    if name == "c3":
        return B.c3(n_pins=4, cells_per_pin=16, n_a=8, outers=1, inner=1), "c3 generator 64x64 cells, n_a=8, 2 groups"
    if name in ("c5", "c5w"):
        return B.c5(n_pins=4, cells_per_pin=16, n_a=4, outers=1, inner=1), "c5 generator 64x64 cells, n_a=4, 7 groups"
    return B.c4(nx=64, blocks=4, n_a=8, cycles=1), "c4 generator at 64x64 cells, n_a=8"


def reference_package():
    """The unmodified reference `convsn`: the driver's offline install under
    baseline/_ref, else the read-only source tree (this container only).  None when
    neither exists (the oracle port stands in)."""
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "convsn")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import convsn
            return convsn, path
    return None, None


def time_reference_cycles(pd, steps, warmup):
    """warmup + steps multigrid iterations of the reference's own driver loop
    (`convsn.eigen._run_cycles`, R/eigen.py:138-156: flux, group source,
    sawtooth_cycle with PGState), one cycle per step; returns (per-cycle seconds,
    kind, where).  Falls back to the oracle port (oracle/) when `convsn` is absent."""
    convsn, where = reference_package()
    times = []
    if convsn is not None:
        from convsn import eigen as re
        from convsn import discretisation as rd
        from convsn.grid import Field
        from convsn.materials import CrossSections
        from convsn.multigrid import PGState
        from convsn.problems import ProblemSpec
        mats = [CrossSections(m.name, m.sigma_a, m.sigma_s, m.nu_sigma_f, m.sigma_f, m.chi)
                for m in pd.materials]
        prob = ProblemSpec(name=pd.name, nx=pd.nx, ny=pd.ny, dx=pd.dx, dy=pd.dy,
                           region_map=pd.region_map, materials=mats, source=pd.source,
                           n_groups=pd.n_groups)
        o = dict(pd.options)
        pg = o.pop("pg", None)
        if pg is not None:
            o["pg"] = rd.PGConfig(**pg)
        opts = re.SolverOptions(**o)
        st = re.setup_transport(prob, opts)
        psi = Field(st.grid, st.quad.n_dir, st.mat.n_groups)
        if st.mat.fissile:            # power iteration's start: psi = 1, production 1
            psi.data[...] = 1.0
        pgs = PGState(opts.k_avg_theta)
        fq = None
        if st.mat.fissile:
            phi = re.scalar_flux(psi, st.quad)
            fq = (st.mat.chi * np.einsum("xyg,xyg->xy", st.mat.nu_sigma_f, phi)[:, :, None])[:, :, None, :]
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            psi, _ = re._run_cycles(psi, st, 1, fission_frozen=fq, pg_state=pgs)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
        return times, "reference", f"convsn {getattr(convsn, '__version__', '')} from {where}".strip()
    import oracle as O      # the port: test infrastructure, the baseline's stand-in only
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _util import oracle_options, oracle_problem
    st = O.setup(oracle_problem(pd), oracle_options(pd))
    data = O.padded(pd.nx, pd.ny, st.h, st.quad.n_dir, pd.n_groups)
    pgs = O.PGState(st.o.k_avg_theta)
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        phi = O.scalar_flux(data, st.h, st.quad.weights)
        q = O.group_source(phi, st.mat)
        O.sawtooth_cycle(data, q, st.levels, st.taps, st.o.order, st.o.pg, st.o.scheme,
                         st.o.jacobi_sweeps, st.o.pg_sweeps, pgs)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    return times, "port", "oracle/convsn_port.py (reference not installed)"


def threads_used():
    return max(int(os.environ.get(v, "0") or 0) for v in CPU_THREAD_VARS) or os.cpu_count()


def run_cpu_sample(config):
    """The cpu_baseline leg (a subprocess of the B200 arm, thread pools pinned before
    numpy loaded): one cycle of the bounded sample; prints one JSON object."""
    pd, desc = cpu_sample_problem(config)
    ts, kind, where = time_reference_cycles(pd, 1, 0)
    print(json.dumps({"value": pd.dof() / ts[0], "unit": "DOF-updates/s",
                      "cores": threads_used(), "kind": kind,
                      "sample": f"{desc}; 1 cycle, {ts[0]:.1f} s; {where}; {cpu_model()}, "
                                f"{threads_used()} thread(s) of {os.cpu_count()} "
                                f"(single-threaded NumPy)"}), flush=True)


def cpu_baseline_start(config):
    """Start the cpu_baseline leg in a subprocess (1 thread, its own core) so it runs
    beside the GPU-side probes; cpu_baseline_result() collects its JSON."""
    env = dict(os.environ, **{v: "1" for v in CPU_THREAD_VARS})
    return subprocess.Popen([sys.executable, os.path.abspath(__file__), "--cpu-sample", config],
                            env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)


def cpu_baseline_result(proc):
    try:
        out, _ = proc.communicate(timeout=600)
        return json.loads(out.strip().splitlines()[-1])
    except (subprocess.SubprocessError, ValueError, IndexError) as e:
        proc.kill()
        return {"value": None, "error": f"cpu baseline failed: {e}"}


def run_reference(args, rank):
    if rank != 0:
        return
    pd, desc = cpu_sample_problem(args.config, arm=True)
    steps, warmup = args.steps, args.warmup
    times, kind, where = time_reference_cycles(pd, steps, warmup)
    dof = pd.dof()
    total = float(sum(times))
    value = dof * len(times) / total
    line = {
        "impl": "reference", "metric": "space-angle DOF-updates/s per sawtooth cycle",
        "value": value, "unit": "DOF-updates/s", "n_gpus": args.gpus, "steps": steps,
        "warmup": warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
        "config": {"workload": f"{args.config} (CPU sample: {desc})", "dof_per_step": dof},
        "cpu_baseline": {"value": value, "unit": "DOF-updates/s", "cores": threads_used(),
                         "kind": kind,
                         "sample": desc + f"; {steps} cycles after {warmup} warm-up; {where}; "
                                          f"{cpu_model()}, {threads_used()} thread(s) of "
                                          f"{os.cpu_count()} (single-threaded NumPy)"},
        "e2e": {"value": value, "unit": "DOF-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 arm
def probe_config(name, dtype_name, steps=4, warmup=2):
    """A few eagerly launched, event-timed cycles of another BASELINE config on this GPU:
    cycle time and the fused sweep's roofline (the p = 1 configs C3 and C5-weak, beside
    the p = 3 headline)."""
    import torch
    import paper_2301_09991_b200 as P
    from paper_2301_09991_b200.eigen import Solver
    from paper_2301_09991_b200.problems import problem_from_data
    pd = workload(name)
    eigen = pd.driver == "power_iteration"
    inner = pd.inner_iters or 1
    opts = options_for(P, pd, dtype_name, None if eigen else steps + warmup)
    if eigen:
        opts.outer_iters = -(-(steps + warmup) // inner)
    solver = Solver(problem_from_data(pd), opts, inner if eigen else None)
    eng = solver.eng
    eng.use_graphs = False
    for _ in range(warmup):
        solver.step()
    eng.probe = {}
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        solver.step()
    ev1.record()
    torch.cuda.synchronize()
    probe = {k: [a.elapsed_time(b) for a, b in v] for k, v in eng.probe.items()}
    ms_k = float(np.mean(probe["pg_sweep"]))
    peak, peak_kind, peaks = measured_peaks()
    esz = 4 if opts.torch_dtype() == torch.float32 else 8
    hbm, fp, bound, roof_frac = sweep_roofline(pd, pd.dof(), esz, eng, ms_k, peak, peak_kind, peaks)
    out = {"workload": WORKLOADS.get(name, name), "dof_per_cycle": pd.dof(),
           "ms_per_cycle": ev0.elapsed_time(ev1) / steps, "cycles": steps,
           "value": pd.dof() * steps / (ev0.elapsed_time(ev1) * 1e-3),
           "pg_sweep": {"ms_per_launch": ms_k, "bound": bound, "hbm_frac": hbm["frac"],
                        "hbm_GBps": hbm["achieved"], "bytes_per_dof": hbm["bytes_per_dof"],
                        "fp32_frac": fp["frac"], "roof_frac": roof_frac},
           "kernels_ms": {k: float(np.mean(v)) for k, v in probe.items()}}
    eng.probe = None
    del solver, eng
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    return out


def run_b200(args, rank, world, local_rank):
    import torch
    import paper_2301_09991_b200 as P
    from paper_2301_09991_b200 import _lib
    from paper_2301_09991_b200.eigen import Solver
    from paper_2301_09991_b200.problems import problem_from_data

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = _lib.load()
    dist = None
    if world > 1:
        import torch.distributed as dist
    pd = workload(args.config, args.nx, world, args.na, args.slabs)
    total = args.warmup + args.steps
    eigen = pd.driver == "power_iteration"
    inner = pd.inner_iters or 1
    opts = options_for(P, pd, args.dtype, None if eigen else total, args.fold)
    if eigen:
        opts.outer_iters = -(-total // inner)
    prob = problem_from_data(pd)
    if world > 1:       # x-slab domain decomposition, NCCL halo exchange (strong scaling)
        from paper_2301_09991_b200.dd import DDSolver, TorchDistComm
        make = lambda: DDSolver(prob, opts, inner if eigen else None, comm=TorchDistComm())
    else:
        make = lambda: Solver(prob, opts, inner if eigen else None)
    solver = make()
    eng = solver.eng
    # whole-cycle CUDA graphs on one GPU only: a DD cycle has NCCL calls and host waits
    # between its launches (DDCycleEngine keeps its own opt-in coarse-solve graphs)
    graphs = world == 1 and (args.graphs == "on" or (args.graphs == "auto"
                                                     and args.config not in ("c4", "c5w")))
    if world == 1:
        eng.use_graphs = graphs
    eng.full_sync = args.full_sync
    if args.pad_delta:             # A/B: sweep through the TMA kernel (padded correction)
        eng.pad_delta = True
    dtype = opts.torch_dtype()
    hist = []
    sampler = ClockSampler(local_rank)
    sampler.start()
    for _ in range(args.warmup):
        hist.append(solver.step())
    # ---- timed region: K cycles, device-timed with CUDA events, clocks sampled
    probe_live = not graphs          # per-kernel events inside the timed region (eager path)
    eng.probe = {} if probe_live else None
    frozen_before = []
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    sampler.mark()
    n_launch0 = lib.csn_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        frozen_before.append(bool(solver.pgs.frozen))
        hist.append(solver.step())
    ev1.record()
    torch.cuda.synchronize()
    n_launch = lib.csn_launch_count() - n_launch0
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64,
                         device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    kernel_timing = "CUDA events around each launch inside the timed region (eager launches)"
    if not probe_live:               # graphs in the timed region: break down in an eager pass
        eng.use_graphs = False
        eng.probe = {}
        extra = make()
        extra.eng.use_graphs = False
        extra.eng.probe = eng.probe
        for _ in range(min(total, args.warmup + 3)):
            extra.step()
        torch.cuda.synchronize()
        kernel_timing = ("CUDA events, eager pass of the first W+3 cycles after the timed "
                         "region (the timed region replays CUDA graphs)")
    probe = {k: [a.elapsed_time(b) for a, b in v] for k, v in (eng.probe or {}).items()}
    eng.probe = None
    dof = pd.dof() // 2 if args.fold else pd.dof()   # DOF actually updated
    value = dof * args.steps / (ms * 1e-3)          # global DOF: strong scaling over ranks
    ldof = dof // world                              # this rank's slab: kernel-level rates

    # ---- roofline of the dominant kernel (fused PG sweep, K5)
    peak, peak_kind, peaks = measured_peaks()
    esz = 4 if dtype == torch.float32 else 8
    kernel_stats = {}
    for k, ts in probe.items():
        kernel_stats[k] = {"ms_avg": float(np.mean(ts)), "launches": len(ts),
                           "ms_min": float(np.min(ts)), "ms_max": float(np.max(ts))}
        if per_dof_bytes(k, esz, eng):
            kernel_stats[k]["GBps"] = per_dof_bytes(k, esz, eng) * ldof / (np.mean(ts) * 1e-3) / 1e9
    dominant = "pg_sweep" if "pg_sweep" in probe else "upwind_residual"
    roof = None
    if dominant in probe:
        ms_k = float(np.mean(probe[dominant]))
        # the committed ncu capture is of the default 1-GPU workload
        traffic = (committed_traffic(args.config, dominant, args.dtype)
                   if world == 1 and not args.fold and args.nx is None and args.na is None
                   else None)
        common = {"kernel": dominant, "traffic": traffic, "ms_per_launch": ms_k,
                  "share_of_step": ms_k * len(probe[dominant]) / (sum(sum(v) for v in probe.values()) or 1),
                  "timing": kernel_timing}
        if dominant == "pg_sweep":
            hbm, fp, bound, roof_frac = sweep_roofline(pd, ldof, esz, eng, ms_k, peak, peak_kind,
                                                       peaks)
            main = fp if bound == "fp32" else hbm
            roof = {"bound": bound, "achieved": main["achieved"], "peak": main["peak"],
                    "unit": main["unit"], "frac": main["frac"], "peak_source": main["peak_source"],
                    **common, "bytes_per_launch": hbm["bytes_per_launch"],
                    "hbm": hbm, "fp32": fp, "roof_frac": roof_frac,
                    "note": ("bound = the lower roof for this ConvFEM order: t_roof = max(bytes / "
                             "measured HBM, flops / FP32 peak); roof_frac = t_roof / launch time")}
        else:
            bpl = per_dof_bytes(dominant, esz, eng) * ldof
            roof = {"bound": "hbm", "achieved": bpl / (ms_k * 1e-3) / 1e9, "peak": peak,
                    "unit": "GB/s", "frac": bpl / (ms_k * 1e-3) / 1e9 / peak,
                    "bytes_per_launch": bpl, **common}
    live = sum(1 for f in frozen_before if not f)
    b_cycle = (bytes_model(pd, solver.setup.hierarchy, True) * live
               + bytes_model(pd, solver.setup.hierarchy, False) * (args.steps - live)) / args.steps
    cycle_roof = b_cycle / (ms / args.steps * 1e-3) / 1e9

    # ---- end to end through the public API with host buffers (rank-local)
    e2e = None
    n_levels, k_hist = solver.setup.hierarchy.n_levels, list(solver.k_history)
    if not args.no_e2e:
        # release the timed solver's device buffers first: the solve below allocates its
        # own through torch's caching allocator, as a fresh call in a running service would
        setup_levels = [l.sigma_t.size for l in solver.setup.hierarchy.levels]
        mf = solver.setup.mat
        del solver, eng
        import gc
        gc.collect()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world > 1:
            res = make().run()
        else:
            res = P.solve_fixed_source(prob, opts) if not eigen else \
                P.power_iteration(prob, opts, inner_iters=inner)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if world > 1:                    # the job's time: the slowest rank
            w = torch.tensor([wall], dtype=torch.float64,
                             device=dev if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(w, op=dist.ReduceOp.MAX)
            wall = float(w.item())
        ncyc = len(res.residual_history)
        h2d = sum(a.nbytes for a in (mf.sigma_s, mf.source, mf.nu_sigma_f, mf.chi))
        h2d += sum(n * esz for n in setup_levels)
        d2h = res.phi.nbytes + 8 * ncyc
        e2e = {"value": dof * ncyc / wall, "unit": "DOF-updates/s",
               "h2d_bytes_per_step": h2d / ncyc, "d2h_bytes_per_step": d2h / ncyc,
               "cycles": ncyc, "wall_s": wall,
               "note": "solve_fixed_source/power_iteration call incl. setup, uploads, phi read-back"}

    # ---- CPU baseline (oracle port, bounded sample, rank 0 at N = 1)
    cpu, cpu_proc = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_proc = cpu_baseline_start(args.config)

    # ---- the p = 1 configs' fused sweep beside the p = 3 headline (1 GPU, default run)
    others = None
    if (rank == 0 and world == 1 and not args.no_extra and args.config == "c4" and args.nx is None
            and args.na is None):
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        others = {}
        for name, steps in (("c3", 10), ("c5w", 4)):
            try:
                others[name] = probe_config(name, args.dtype, steps=steps, warmup=2)
            except Exception as e:   # e.g. not enough free memory: say so, keep the line
                others[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if cpu_proc is not None:
        cpu = cpu_baseline_result(cpu_proc)

    if rank == 0:
        line = {
            "metric": "space-angle DOF-updates/s per sawtooth cycle",
            "value": value, "unit": "DOF-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.config == "c5w" else "strong", "vs_baseline": None,
            "dtype": "f32" if dtype == torch.float32 else "f64",
            "data": "synthetic (seeded BASELINE generators, paper_2301_09991_b200/benchmarks.py)",
            "config": {"workload": f"{args.config}: " + WORKLOADS.get(args.config, ""),
                       "dof_per_cycle": dof, "nx": pd.nx, "ny": pd.ny,
                       "ordinates": 8 * pd.n_a ** 2, "groups": pd.n_groups,
                       "fold_z": bool(args.fold),
                       "order": pd.options["order"], "scheme": pd.options["scheme"],
                       "levels": n_levels, "live_cycles": live,
                       "frozen_cycles": args.steps - live, "cuda_graphs": graphs,
                       **({"tuning": list(args.tune)} if args.tune else {}),
                       "l2": "per-cycle fields >> 126 MB L2 (no flush needed)"
                       if dof * esz > 4 * 126e6 else "fields partly L2-resident; see DESIGN.md",
                       "parallelism": (f"x-slab domain decomposition over {world} GPUs "
                                       f"(NCCL halo exchange, gathered coarse levels)")
                       if world > 1 else "1 GPU"},
            "roofline": roof,
            "cycle_roofline": {"bytes_per_cycle": b_cycle, "achieved": cycle_roof, "peak": peak,
                               "unit": "GB/s", "frac": cycle_roof / peak},
            "kernels": kernel_stats,
            "other_configs": others,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(n_launch),
            "clocks": clocks,
            "residual_history": hist,
        }
        if eigen:
            line["k_history"] = k_hist
        print(json.dumps(line), flush=True)


WORKLOADS = {
    "c4": "1 group, cubic PG, 512x512 cells, 2048 ordinates (n_a=16), 32x32 seeded blocks",
    "c2": "1 group, quadratic PG, 128x128 cells, 512 ordinates, 8x8 seeded blocks",
    "c1": "1 group, linear, PG off (alpha_r=0), 64x64, 128 ordinates",
    "c3": "2-group k-eigenvalue, linear PG, 256x256, 512 ordinates, 5 cycles per outer",
    "c5w": "7-group k-eigenvalue, linear PG, 512x512 cells per GPU stacked along x "
           "((512 N) x 512 global), 2048 ordinates, 3 cycles per outer (weak scaling)",
    "c5": "7-group k-eigenvalue, linear PG, 1024x1024, 2048 ordinates, 64x64 seeded pin "
          "lattice, 3 cycles per outer (strong scaling, >= 4 GPUs)",
}


def committed_traffic(config, kernel, dtype):
    """dram read+write bytes per launch of `kernel` from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(f"{config}:{kernel}:{dtype}")
    except (OSError, ValueError):
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=17)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--nx", type=int, default=None, help="override the cell count (c4 only)")
    ap.add_argument("--na", type=int, default=None,
                    help="override n_a (c4, c5, c5w; plumbing checks, not a BASELINE config)")
    ap.add_argument("--slabs", type=int, default=None,
                    help="c5w: the weak problem of this many ranks, (512 S) x 512, on any world")
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the C3 / C5-weak sweep probes after the headline")
    ap.add_argument("--fold", action="store_true",
                    help="z-mirror fold (half the ordinates, same flux); value counts the "
                         "DOF actually updated, not the full-sphere equivalent")
    ap.add_argument("--graphs", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--full-sync", action="store_true",
                    help="A/B: the host waits for the whole cycle instead of its residual")
    ap.add_argument("--pad-delta", action="store_true",
                    help="A/B: padded finest correction, so the sweep runs in the TMA kernel")
    ap.add_argument("--tune", action="append", default=[], metavar="KEY=VALUE",
                    help="kernel-variant switch (csn_set_tuning), for A/B timing")
    ap.add_argument("--cpu-sample", default=None, metavar="CONFIG",
                    help="internal: the cpu_baseline leg (one reference cycle, 1 thread)")
    args = ap.parse_args()
    if args.cpu_sample:
        run_cpu_sample(args.cpu_sample)
        return
    if args.warmup < 0 or args.steps < 1:
        raise SystemExit("need --steps >= 1")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # CSN_DIST_BACKEND=gloo: plumbing check of the N > 1 path on fewer GPUs than ranks
        # (bands staged through the host; never a performance number)
        backend = os.environ.get("CSN_DIST_BACKEND", "nccl")
        if backend == "gloo":
            local_rank %= torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        dist.init_process_group(backend)
    if args.tune:
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from paper_2301_09991_b200 import _lib
        for kv in args.tune:
            k, v = kv.split("=")
            _lib.set_tuning(k, int(v))
    run_b200(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
