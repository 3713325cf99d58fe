#!/usr/bin/env python
"""IB spread + interpolate benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one scalar spread of 2^20 forces at the predicted positions X*
plus one scalar interpolation of a 256^3 field at X^n (BASELINE config 2,
the configuration the metric is quoted on), on the periodic MAC z-grid
(alpha = (1/2, 1/2, 0)) with the 4-point cosine kernel, FP64.
metric = Lagrangian points / s.  Inputs are synthetic (ib::bench::
scatter_points, seed 1; X* = X^n + U[-0.1h, 0.1h]^3).

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA
events on the operators' stream with a 256 MiB L2 flush between steps
(outside the events); barrier + synchronize on both sides; max over ranks.
Under torchrun (N > 1) the grid is 256 x 256 x 256N, split in z-slabs, one
per GPU, each holding 2^20 points (weak scaling, the same load per GPU as
config 2); every step runs the slab spread with its NCCL ghost-plane sum and
the halo fill + slab interpolation (paper_2012_06646_b200/slab.py).

--impl reference times the reference's own OpenMP CPU path (ib::spread_fused
+ ib::interpolate compiled from the reference headers into oracle/_ref) on
all host threads, same workload and metric; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Lagrangian points/sec for spread+interpolate per step, %HBM roofline, 1/2/4/8 B200"
UNIT = "points/s"
WORKLOAD = ("config 2: 2^20 uniform random points (scatter_points seed 1) on a 256^3 periodic "
            "grid, 4-point cosine (Peskin 2002) kernel, one scalar spread (at X*) + one scalar "
            "interpolation (at X^n) per step, FP64")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-graph", action="store_true", help="time eager launches, not a CUDA graph")
    ap.add_argument("--mac-steps", type=int, default=5, help="MAC vector step timing (0: skip)")
    ap.add_argument("--f32-steps", type=int, default=10,
                    help="FP32 storage-mode step timing, a secondary figure (0: skip)")
    ap.add_argument("--no-serial", action="store_true", help="reference arm: skip the spread_serial timing")
    ap.add_argument("--transport", default="peer", choices=["peer", "collective"],
                    help="N > 1: slab exchange over peer memory (C ABI, one CUDA graph per step) "
                         "or torch.distributed send/recv between graph replays")
    ap.add_argument("--strong", action="store_true",
                    help="N > 1: strong scaling -- config 2 (2^20 points, one 256^3 grid) split into N z-slabs")
    ap.add_argument("--workload", default="c2", choices=["c2", "c1", "w128", "w256", "rbc", "clustered"],
                    help="one-GPU workload (default: BASELINE config 2, the headline)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _affinity() -> set:
    try:
        return set(os.sched_getaffinity(0))
    except Exception:
        return set(range(os.cpu_count() or 1))


# Read once at import, before libgomp (the reference arm) binds the main
# thread to one place and shrinks the mask.
_CPUS = _affinity()


def host_threads() -> int:
    """Host threads available to this process: the reference's OpenMP team
    (workers = nproc), one thread per logical CPU of the
    affinity mask."""
    return max(1, len(_CPUS))


def physical_cores() -> int | None:
    """Distinct physical cores behind the affinity mask (sysfs topology), or
    None when the topology is not readable."""
    try:
        cpus = _CPUS
        cores = set()
        for c in cpus:
            base = f"/sys/devices/system/cpu/cpu{c}/topology/"
            with open(base + "physical_package_id") as f:
                pkg = f.read().strip()
            with open(base + "core_id") as f:
                core = f.read().strip()
            cores.add((pkg, core))
        # A VM that exposes no core topology reports every CPU as core 0.
        return len(cores) if len(cores) > 1 or len(cpus) == 1 else None
    except Exception:
        return None


def omp_env() -> None:
    """Pin the reference's OpenMP team before libgomp initialises."""
    os.environ["OMP_PLACES"] = "cores"
    os.environ["OMP_PROC_BIND"] = "close"
    os.environ["OMP_NUM_THREADS"] = str(host_threads())


def bench_config(workload: str, n: int, grid) -> dict:
    """The config dict both arms print (the driver compares them)."""
    return {"workload": workload, "n_points": int(n), "grid": [int(v) for v in grid]}


def lib_build_id() -> str:
    """Source hash of libibcuda.so (_build.source_id): stamps measured ncu traffic."""
    from paper_2012_06646_b200 import _build

    return _build.source_id()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int, period: float = 0.001):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def sample_now(self):
        """One sample from the calling thread (the timed loop calls this
        between steps -- host side only, outside every event pair -- so the
        region has samples even when the launch loop starves the thread)."""
        if not self.ok:
            return
        nv = self.nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if mask & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self.sample_now()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_reference_steps(data, steps, warmup, threads):
    """Reference ib::spread_fused + ib::interpolate (oracle/_ref), per-step seconds."""
    import numpy as np

    import oracle as O

    N = data["N"]
    g = O.make_grid([N] * 3, data["h"], [0.5, 0.5, 0.0], [1, 1, 1])
    omp_env()
    ts, ti = O.ref_time_step(g, data["x_star"], data["values"], data["x_n"], data["field"],
                             threads, warmup + steps)
    return (np.asarray(ts) + np.asarray(ti))[warmup:]


def workload_name(w: str, n: int, N: int) -> str:
    return WORKLOAD if w == "c2" else (
        f"SURVEY 8(d) workload {w}: {n} points on a {N}^3 periodic grid, one scalar spread "
        "(at X*) + one scalar interpolation (at X^n) per step, FP64")


def run_config(args, world: int, n1: int, N: int) -> dict:
    """The workload a run of `world` ranks measures (both arms print it)."""
    if world == 1:
        return bench_config(workload_name(args.workload, n1, N), n1, [N] * 3)
    if args.strong:
        return bench_config(
            f"config 2, strong scaling: 2^20 points on one 256^3 periodic grid split into {world} "
            "z-slabs, each rank the points homed in its slab; per step one scalar spread (local + "
            "ghost-plane sum) and one scalar interpolation (halo fill + local gather), FP64",
            1 << 20, [256, 256, 256])
    if args.workload == "w256":
        return bench_config(
            f"config 3 (1 point per cell) at constant load, weak scaling: {world} z-slabs of a "
            f"256 x 256 x {256 * world} periodic grid, 256^3 points homed in each slab; per step "
            "one scalar spread (local + ghost-plane sum) and one scalar interpolation (halo fill "
            "+ local gather), FP64", world * 256 ** 3, [256, 256, 256 * world])
    return bench_config(
        f"config 2 per GPU, weak scaling: {world} z-slabs of a 256 x 256 x {256 * world} periodic "
        "grid, 2^20 points homed in each slab; per step one scalar spread (local + ghost-plane "
        "sum) and one scalar interpolation (halo fill + local gather), FP64",
        world << 20, [256, 256, 256 * world])


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    import oracle as O
    from paper_2012_06646_b200 import synth

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libibref.so not built (reference headers absent at build)"}))
        return
    data = synth.survey_config(args.workload)
    threads = host_threads()
    # One step of the full workload takes ~1-2 s on 8 cores: bound the run to a
    # few minutes by capping the number of measured steps.
    steps = min(args.steps, 20)
    warm = min(args.warmup, 1)
    t = cpu_reference_steps(data, steps, warm, threads)
    per = float(statistics.median(t))
    value = data["n"] / per
    # also ib::spread_serial (Alg. 2) at one worker, one call.
    serial_ms = None
    if not args.no_serial:
        import oracle as O

        N = data["N"]
        g = O.make_grid([N] * 3, data["h"], [0.5, 0.5, 0.0], [1, 1, 1])
        t0 = time.perf_counter()
        O.ref_spread(g, data["x_star"], data["values"], algo="serial", workers=1)
        serial_ms = (time.perf_counter() - t0) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(t), "warmup": warm, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": run_config(args, world, data["n"], data["N"]),
        "parallelism": f"OpenMP, {threads} threads (all logical CPUs of the affinity mask; "
                       f"{physical_cores()} physical cores), OMP_PLACES=cores, OMP_PROC_BIND=close "
                       "(rank 0 only)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "physical_cores": physical_cores(), "kind": "reference",
                         "sample": f"{len(t)} full {args.workload} steps ({data['n']} points, "
                                   f"{data['N']}^3{', one slab of the run' if world > 1 else ''}), "
                                   "median"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "spread_serial_1_thread_ms": serial_ms,
    }
    print(json.dumps(line))


def shim_e2e(N: int, n: int, reps: int) -> dict | None:
    """ib::spread_fused + ib::interpolate through include/ib_b200 on pageable
    std::vector buffers (tools/shim_step): the two calls back to back (value)
    and from two host threads (concurrent_value); the caller keeps large
    blocks on the glibc heap so each returned 134 MB GridField reuses pages."""
    import subprocess

    from paper_2012_06646_b200 import _build

    exe = _build.SHIM_STEP
    if not exe.exists():
        return None
    out = {"unit": UNIT, "note": "ib::spread_fused (ws.run_count read) + ib::interpolate through "
                                 "the C++ drop-in include/ib_b200, std::vector (pageable) "
                                 "buffers, results returned by value as in the reference, "
                                 "glibc large blocks kept on the heap (mallopt), "
                                 "tools/shim_step.cpp, wall clock median"}
    for conc, key in ((0, "value"), (1, "concurrent_value")):
        r = subprocess.run([str(exe), str(N), str(n), str(max(reps, 3)), str(conc), "1"],
                           capture_output=True, text=True, timeout=600)
        if r.returncode != 0 or "step_s_median" not in r.stdout:
            return {"unavailable": (r.stdout + r.stderr)[-200:]}
        out[key] = n / float(r.stdout.split()[1])
    return out


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2012_06646_b200 import ib, synth
    from paper_2012_06646_b200.device import DeviceOperators, capture_graph
    from paper_2012_06646_b200.slab import SlabDecomposition

    world, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())  # >1 rank per GPU only in dev runs
    if world > 1:
        backend = os.environ.get("IBC_BENCH_BACKEND", "nccl")  # gloo: dev runs on one GPU
        dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)}
                                            if backend == "nccl" else {}))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    # N = 1: BASELINE config 2 on one grid.  N > 1: the same load per GPU as
    # z-slabs of a 256 x 256 x 256N periodic grid (weak scaling), with the
    # ghost-plane sum and halo fill over NCCL between ring neighbours.
    if world == 1:
        data = synth.survey_config(args.workload)
        n, N, h = data["n"], data["N"], data["h"]
        grid = ib.StaggeredGrid([N] * 3, h, [0.5, 0.5, 0.0], [True] * 3)
        ops = DeviceOperators(local)
        dec = None
    elif args.strong:
        # the one config-2 workload, each rank taking
        # the spread points (X*) and interpolation points (X^n) homed in its
        # z-slab of the 256^3 grid and its owned planes of the field.
        from paper_2012_06646_b200.slab import home_planes, owner_of_planes, slab_bounds

        data = dict(synth.survey_config("c2"))
        n_total, N, h = data["n"], data["N"], data["h"]
        grid = ib.StaggeredGrid([N] * 3, h, [0.5, 0.5, 0.0], [True] * 3)
        ops = DeviceOperators(local)
        dec = SlabDecomposition(grid, rank, world, ops=ops)

        def mine(a):
            t = torch.tensor(np.ascontiguousarray(a), device=dev)
            return (owner_of_planes(home_planes(grid, t, ops), N, world) == rank).cpu().numpy()

        ms, mn = mine(data["x_star"]), mine(data["x_n"])
        zb = slab_bounds(N, world)
        data.update(x_star=np.ascontiguousarray(data["x_star"][ms]),
                    values=np.ascontiguousarray(data["values"][ms]),
                    x_n=np.ascontiguousarray(data["x_n"][mn]),
                    field=np.ascontiguousarray(
                        np.asarray(data["field"]).reshape(N, N * N)[zb[rank]:zb[rank + 1]].reshape(-1)))
        n = len(data["x_n"])
    else:
        data = synth.slab_config(rank, world, 256 ** 3 if args.workload == "w256" else 1 << 20)
        n, N, h = data["n"], data["N"], data["h"]
        grid = ib.StaggeredGrid([N, N, data["nz_global"]], h, [0.5, 0.5, 0.0], [True] * 3)
        ops = DeviceOperators(local)
        dec = SlabDecomposition(grid, rank, world, ops=ops)
    strong = world > 1 and args.strong
    total_points = n_total if strong else world * n
    xs = torch.tensor(data["x_star"], device=dev)
    xn = torch.tensor(data["x_n"], device=dev)
    gv = torch.tensor(data["values"], device=dev)
    fe = torch.tensor(data["field"], device=dev)
    ell = torch.empty(N ** 3, dtype=torch.float64, device=dev)
    E = torch.empty(n, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    transport = args.transport if dec is not None else None
    if dec is not None:
        local_out = torch.empty(dec.local.point_count(), dtype=torch.float64, device=dev)
        field_local = torch.empty(dec.local.point_count(), dtype=torch.float64, device=dev)
        # Size every scratch buffer before any cross-rank handshake.
        dec._device_spread(xs, gv, out=local_out)
        dec._device_interpolate(field_local, xn, out=E)
        torch.cuda.synchronize()
        dist.barrier()
        if transport == "peer":
            # Peer-memory exchange: CUDA IPC handles swapped once over the
            # process group; the field's owned planes live in the shared slab.
            peer = dec.use_peer_transport()
            peer.owned_field.copy_(fe)
            torch.cuda.synchronize()
            dist.barrier()
    # The device-side pieces of a step: both operators on one GPU; for slabs
    # the local spread, the ghost-plane sum, the halo fill and the local
    # gather -- one piece over peer memory (the whole step is one CUDA graph),
    # or the local operators with the NCCL exchanges between them (eager:
    # they go through torch.distributed).
    launch_counters = [ops]
    if dec is None:
        # The two operators are independent (X* vs X^n): X^n is binned on a
        # second stream and context while the spread runs (its sort kernels
        # leave room beside the spread's), the gather follows the spread
        # sweep (the two shared-memory sweeps do not share SMs well).
        ops_b = DeviceOperators(local)
        launch_counters.append(ops_b)
        side = torch.cuda.Stream(dev)
        binned = [None]

        def pair():
            main = torch.cuda.current_stream(dev)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                binned[0] = ops_b.bin_points(xn, grid, binned=binned[0])
            ops.spread(xs, gv, grid, out=ell)
            main.wait_stream(side)
            ops_b.interpolate_binned(fe, binned[0], out=E)

        local_ops = [pair]
        # per-kernel-class device times: the two operators one after the other
        profile_ops = [lambda: (ops.spread(xs, gv, grid, out=ell), ops.interpolate(fe, xn, grid, out=E))]
    elif transport == "peer":
        local_ops = [lambda: (dec.spread(xs, gv), dec.interpolate(None, xn, out=E))]
    else:
        local_ops = [lambda: dec._device_spread(xs, gv, out=local_out),
                     lambda: dec._device_interpolate(field_local, xn, out=E)]
    graphs = [None] * len(local_ops)

    if dec is not None:
        profile_ops = local_ops

    def step(eager=False, profile=False):
        def run(k):
            if profile:
                profile_ops[k]()
            elif graphs[k] is not None and not eager:
                graphs[k].replay()
            else:
                local_ops[k]()

        run(0)
        if dec is not None and transport != "peer":
            dec.ghost_sum(local_out)
            dec.halo_fill(fe, out=field_local)
            run(1)

    for i in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l0 = sum(o.launches for o in launch_counters)
    step()
    torch.cuda.synchronize()
    launches_per_step = sum(o.launches for o in launch_counters) - l0
    # Every kernel and memset of the operators is captured once in a CUDA
    # graph and replayed (the pipeline has no host round trip).
    if not args.no_graph:
        for k, f in enumerate(local_ops):
            graphs[k] = capture_graph(f)
        step()
        torch.cuda.synchronize()
    graph = graphs[0]

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(K):
            flush.fill_(float(i))  # evict L2 (256 MiB > 126 MB) outside the events
            ev[i][0].record()
            step()
            ev[i][1].record()
            clk.sample_now()
        torch.cuda.synchronize()
    launches = launches_per_step * K  # our kernels per step (graph replays launch them all)
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / K
    value = total_points * K / (total_ms * 1e-3)

    # Per-kernel-class device times (CUDA events on the operators' stream), separate pass.
    P = max(3, min(K, 10))
    ops.context.set_profiling(True)
    ops.context.reset_profile()
    for i in range(P):
        flush.fill_(float(i))
        step(eager=True, profile=True)  # per-kernel-class events: eager launches, one stream
    prof = ops.context.profile()
    ops.context.set_profiling(False)
    per_launch = {k[:-3]: prof[k] / P * 1e3 for k in prof if k.endswith("_ms")}  # us per step
    n_omega = dec.lay.nloc * N * N if dec is not None else N ** 3  # grid points this rank owns
    alg = {"spread": 32 * n + 8 * n_omega, "interp": 32 * n + 8 * n_omega}
    dom = max(("spread", "interp"), key=lambda k: per_launch.get(k, 0.0))
    peak, peak_src = peaks()
    achieved = alg[dom] / (per_launch[dom] * 1e-6) / 1e9
    # dram bytes per launch from `ncu --set full` of this very build (profiles/
    # traffic.json, written by tools/traffic.py); null when the build differs.
    traffic, traffic_src = None, "no ncu capture of this build"
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            tj = json.loads(tf.read_text())
            if tj.get("build") == lib_build_id() and tj.get("workload") == args.workload:
                traffic = tj.get(dom)
                traffic_src = f"ncu --set full, profiles/traffic.json (build {tj['build']})"
        except Exception:
            traffic = None
    step_bytes = 64 * n + 16 * n_omega

    # End to end through the public API: pinned host buffers in, results out.
    e2e = None
    if args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hx_s, hx_n, hg, hf = pin(data["x_star"]), pin(data["x_n"]), pin(data["values"]), pin(data["field"])
        h_ell = torch.empty(n_omega, dtype=torch.float64).pin_memory()
        h_E = torch.empty(n, dtype=torch.float64).pin_memory()
        if dec is None:
            # The reference-facing C ABI with host buffers (ibc_spread /
            # ibc_interpolate: copies in, operator, copy out, synchronous) --
            # the call ib::spread_fused / ib::interpolate make through
            # include/ib_b200/ib.hpp -- on pinned host memory.
            import ctypes as C

            from paper_2012_06646_b200 import _capi

            lib = _capi.load()
            ctx = ib.default_context(local)
            ws = ib.SpreadWorkspace(n, grid, context=ctx)
            vp = lambda t: C.c_void_p(t.data_ptr())

            from concurrent.futures import ThreadPoolExecutor

            pool = ThreadPoolExecutor(max_workers=1)

            def spread_call():
                _capi.check(lib.ibc_spread(ctx.handle, C.byref(grid.c_grid), _capi.IBC_KERNEL_COSINE4,
                                           _capi.IBC_SPREAD_FUSED, vp(hx_s), vp(hg), n, n, 0,
                                           ws.handle, 0, vp(h_ell)))

            def interp_call():
                _capi.check(lib.ibc_interpolate(ctx.handle, C.byref(grid.c_grid),
                                                _capi.IBC_KERNEL_COSINE4, vp(hf), vp(hx_n), n, 0,
                                                vp(h_E)))

            def e2e_step():
                # The two calls of a step are independent (X* and X^n): the
                # interpolation runs on a second host thread (ctypes releases
                # the GIL), each call on its own lane of the context, so the
                # spread's grid copy-out overlaps the interpolation's field
                # copy-in on the two PCIe directions.
                fut = pool.submit(interp_call)
                spread_call()
                fut.result()

            def e2e_sequential():
                spread_call()
                interp_call()
            note = ("ibc_spread(FUSED) and ibc_interpolate through the C ABI with pinned host "
                    "buffers (H2D + operator + D2H inside each call), the two calls issued "
                    "concurrently from two host threads, wall clock, median")
        else:
            def e2e_step():
                d_xs, d_g = hx_s.to(dev, non_blocking=True), hg.to(dev, non_blocking=True)
                d_xn, d_f = hx_n.to(dev, non_blocking=True), hf.to(dev, non_blocking=True)
                h_ell.copy_(dec.spread(d_xs, d_g), non_blocking=True)
                h_E.copy_(dec.interpolate(d_f, d_xn), non_blocking=True)
                torch.cuda.synchronize()
            note = "SlabDecomposition.spread + .interpolate with H2D inputs / D2H outputs (pinned), wall clock, median, max over ranks"
        for _ in range(2):  # warm-up: lanes, staging, pinned-memory registrations
            e2e_step()
        torch.cuda.synchronize()
        ts = []
        for i in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        e2e_s = statistics.median(ts)
        if world > 1:
            t = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": total_points / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(hx_s.nbytes + hg.nbytes + hx_n.nbytes + hf.nbytes),
               "d2h_bytes_per_step": int(n_omega * 8 + n * 8), "note": note}
        if dec is None:
            # Same calls back to back on one thread, and through the C++
            # drop-in on pageable std::vector buffers (tools/shim_step.cpp).
            ts = []
            for i in range(args.e2e_steps):
                t0 = time.perf_counter()
                e2e_sequential()
                ts.append(time.perf_counter() - t0)
            e2e["sequential"] = {"value": total_points / statistics.median(ts), "unit": UNIT,
                                 "note": "same two calls back to back on one thread"}
            e2e["shim"] = shim_e2e(N, n, args.e2e_steps)

    # Secondary figure: the reference's MAC vector step -- 6
    # interpolations + 3 spreads on the three component grids + tether forces
    # and position updates -- device-resident (step.py), same n and N,
    # captured in a CUDA graph like the headline step.
    mac = None
    if world == 1 and args.mac_steps > 0:
        from paper_2012_06646_b200.step import MacStepLoop, StepConfig

        loop = MacStepLoop(StepConfig(refinement=N, point_count=n), device=local, ops=ops,
                           points=data["x_n"])
        for _ in range(2):
            loop.step()
        torch.cuda.synchronize()
        mgraph = None
        if not args.no_graph:
            mgraph = capture_graph(loop.step)
            mgraph.replay()
            torch.cuda.synchronize()
        mev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.mac_steps)]
        for i in range(args.mac_steps):
            flush.fill_(float(i))
            mev[i][0].record()
            if mgraph is not None:
                mgraph.replay()
            else:
                loop.step()
            mev[i][1].record()
        torch.cuda.synchronize()
        mac_ms = sum(a.elapsed_time(b) for a, b in mev) / args.mac_steps
        mac = {"value": n / (mac_ms * 1e-3), "unit": UNIT, "ms_per_step": mac_ms,
               "steps": args.mac_steps,
               "workload": "ib::bench::run_benchmark step on the MAC grids (alpha = (0,.5,.5), "
                           "(.5,0,.5), (.5,.5,0)) of the same 256^3 periodic cube, fixed shear "
                           "field, tether forces: 2 x interpolate_vector + 1 x spread_vector + "
                           "updates per step, same 2^20 points, FP64, CUDA graph"}
        del loop

    # Secondary figure: the same step in the FP32 storage mode (ibc_*_f32:
    # float points / values / fields / results, FP64 arithmetic inside).
    f32 = None
    if world == 1 and args.f32_steps > 0 and dec is None:
        xs32, gv32, fe32, xn32 = xs.float(), gv.float(), fe.float(), xn.float()
        ell32 = torch.empty(n_omega, dtype=torch.float32, device=dev)
        E32 = torch.empty(n, dtype=torch.float32, device=dev)
        binned32 = [None]

        def f32_op():  # the headline step's schedule (X^n binned beside the spread)
            main = torch.cuda.current_stream(dev)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                binned32[0] = ops_b.bin_points(xn32, grid, binned=binned32[0])
            ops.spread(xs32, gv32, grid, out=ell32)
            main.wait_stream(side)
            ops_b.interpolate_binned(fe32, binned32[0], out=E32)
        for _ in range(3):
            f32_op()
        torch.cuda.synchronize()
        fgraph = None if args.no_graph else capture_graph(f32_op)
        fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.f32_steps)]
        for i in range(args.f32_steps):
            flush.fill_(float(i))
            fev[i][0].record()
            fgraph.replay() if fgraph is not None else f32_op()
            fev[i][1].record()
        torch.cuda.synchronize()
        f32_ms = sum(a.elapsed_time(b) for a, b in fev) / args.f32_steps
        f32_bytes = 32 * n + 8 * n_omega
        f32 = {"value": n / (f32_ms * 1e-3), "unit": UNIT, "ms_per_step": f32_ms,
               "steps": args.f32_steps, "dtype": "f32 storage, f64 arithmetic",
               "step_roofline": {"alg_bytes": f32_bytes,
                                 "frac": f32_bytes / (f32_ms * 1e-3) / 1e9 / peak},
               "workload": "the headline step with float points, values, field and results "
                           "(ibc_spread_device_f32, ibc_bin_points_device_f32 + "
                           "ibc_interpolate_binned_device_f32), same schedule, CUDA graph"}
        del xs32, gv32, fe32, xn32, ell32, E32, binned32

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # The reference arm in a child process (its OpenMP team pinned there),
        # a bounded sample of the same workload.
        import subprocess

        try:
            r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                                "--workload", args.workload, "--steps", "2", "--warmup", "1",
                                "--no-serial"], capture_output=True, text=True, timeout=900)
            ref = json.loads(r.stdout.strip().splitlines()[-1])
            cpu = dict(ref["cpu_baseline"])
            cpu["sample"] = f"2 full {args.workload} steps (ib::spread_fused + ib::interpolate, " \
                            "oracle/_ref, OpenMP) after 1 warm-up, median, in a child process"
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": run_config(args, world, n if world == 1 else total_points, N),
            "parallelism": (f"z-slab x{world} (ghost-plane sum + halo fill over "
                            + ("NVLink peer memory, one CUDA graph per step)" if transport == "peer"
                               else "torch.distributed send/recv)"))
                           if world > 1 else "single GPU",
            "n_points_per_gpu": n,
            "l2": "flushed between steps (256 MiB write outside the events)",
            "cuda_graph": graph is not None,
            "step_streams": ("X^n binned on a second stream beside the spread (ibc_bin_points_device), "
                             "the gather after the spread sweep (ibc_interpolate_binned_device)"
                             if world == 1 else "one stream per rank"),
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "alg_bytes_per_launch": alg[dom], "launch_us": per_launch[dom]},
            "step_roofline": {"alg_bytes": step_bytes,
                              "achieved": step_bytes / (ms_per_step * 1e-3) / 1e9,
                              "frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / peak},
            "breakdown_us": {k: round(v, 2) for k, v in per_launch.items()},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "mac_vector_step": mac,
            "f32_storage_step": f32,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        omp_env()  # before libgomp initialises: the reference's OpenMP team, pinned to cores
        run_reference(args)
    else:
        # Not pinned: OMP_PROC_BIND would bind this process's main thread (and
        # every host thread it starts: the e2e callers, the staging copies) to
        # one core.  The in-run CPU baseline runs in its own process.
        run_ours(args)


if __name__ == "__main__":
    main()
