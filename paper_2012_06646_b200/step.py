"""Device-resident MAC step loop -- the reference's bench step on the GPU.

Restates `ib::bench::run_benchmark` (`inc/bench/run.hpp:59-128`) with the
data resident in HBM: per step

  (a) u* = interpolate_vector(u, X^n)        -- 3 interpolations
  (b) X* = X^n + dt u*
  (c) F  = hookean_force(X*, X0)             -- minimal-image tether, setup.hpp:58-74
  (d) l  = spread_vector(X*, F)              -- 3 spreads (kept, not fed back)
  (e) u' = interpolate_vector(u, X^n)        -- 3 interpolations (== u*)
  (f) X^{n+1} = X^n + dt u'

on the MAC component grids of `mac_grids` (`setup.hpp:16-23`, staggering 0
along the component's own axis, 1/2 along the others) with the fixed shear
field of `shear_field` (`setup.hpp:27-40`).  The six interpolations and three
spreads run through libibcuda's device operators -- the three components of
a vector operation concurrently, each on its own stream and context -- and
the per-point updates (b), (c), (f) are a few elementwise torch ops on (n, 3)
tensors (plumbing around the operators, as the reference's loops are around
its calls).

Steps (a) and (e) interpolate the same field at the same points, so each
component's points are binned once per step (`DeviceOperators.bin_points`,
ibc_bin_points_device) and both gathers reuse the binning.  `run_benchmark`
times each vector operation on the device and returns the reference's
`TimingReport` fields; `write_csv` writes the reference's CSV schema
(`report.hpp:16-18, 50-66`) and `fnv1a` the physics fingerprint
(`run.hpp:44-52, 120-126`).

This is SURVEY.md 8(f) item 2 and the "MAC vector step" secondary figure of
8(d); the headline metric stays the scalar spread + interpolation pair.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .ib import StaggeredGrid


@dataclass
class StepConfig:
    """ib::bench::BenchmarkConfig (`inc/bench/config.hpp:15-31`) defaults."""

    refinement: int = 64
    point_count: int = 1 << 16
    domain_edge_um: float = 16.0
    dt_us: float = 0.1
    shear_rate: float = 1000.0       # 1/s
    spring_constant: float = 0.01    # dyn/cm
    seed: int = 1
    steps: int = 100
    workers: int = 1                  # accepted for the CSV; the device picks its own
    sweep_width: int = 8
    algorithm: str = "fused"

    @property
    def edge_cm(self) -> float:
        return self.domain_edge_um * 1e-4

    @property
    def dt_s(self) -> float:
        return self.dt_us * 1e-6


def mac_grids(refinement: int, edge_cm: float) -> list[StaggeredGrid]:
    """ib::bench::mac_grids (setup.hpp:16-23)."""
    h = edge_cm / refinement
    ext = [refinement] * 3
    return [StaggeredGrid(ext, h, st, [True] * 3)
            for st in ([0.0, 0.5, 0.5], [0.5, 0.0, 0.5], [0.5, 0.5, 0.0])]


def shear_field(grids, shear_rate: float, edge_cm: float, device):
    """ib::bench::shear_field (setup.hpp:27-40): u = (0, 0, rate (y - L/2)) on
    the component grids, colex order (x fastest)."""
    import torch

    g = grids[2]
    nx, ny, nz = g.extents
    iy = torch.arange(ny, dtype=torch.float64, device=device)
    y = g.spacing() * (iy + g.staggerings[1])
    row = shear_rate * (y - 0.5 * edge_cm)                       # per y
    w = row.view(1, ny, 1).expand(nz, ny, nx).contiguous().view(-1)
    zero = lambda gg: torch.zeros(gg.point_count(), dtype=torch.float64, device=device)
    return [zero(grids[0]), zero(grids[1]), w]


def hookean_force(predicted, anchors, k: float, edge_cm: float, out=None):
    """ib::bench::hookean_force (setup.hpp:58-74): F = -k d, d the minimal
    image of X* - X0 on the periodic cube.  (n, 3) in -> (3, n) out."""
    import torch

    d = predicted - anchors
    d = d - edge_cm * torch.round(d / edge_cm)
    f = (-k * d).t()
    if out is None:
        return f.contiguous()
    out.copy_(f)
    return out


class MacStepLoop:
    """The reference bench step with every array on one GPU."""

    def __init__(self, cfg: StepConfig, device: int = 0, ops=None, points=None,
                 concurrent: bool = True):
        import numpy as np
        import torch

        from . import synth
        from .device import DeviceOperators

        self.cfg = cfg
        self.dev = torch.device("cuda", device)
        self.ops = ops or DeviceOperators(device)
        # The three components are independent: with `concurrent`, each runs
        # on its own stream and context (its own scratch), forked from and
        # joined back to the caller's stream -- graph-capturable.
        self.concurrent = concurrent
        if concurrent:
            self.comp_ops = [self.ops] + [DeviceOperators(device) for _ in range(2)]
            self.streams = [torch.cuda.Stream(self.dev) for _ in range(3)]
        else:
            self.comp_ops = [self.ops] * 3
            self.streams = None
        L = cfg.edge_cm
        self.grids = mac_grids(cfg.refinement, L)
        self.velocity = shear_field(self.grids, cfg.shear_rate, L, self.dev)
        pts = points if points is not None else synth.scatter_points(cfg.point_count, L, cfg.seed)
        self.X = torch.tensor(np.ascontiguousarray(pts, dtype=np.float64), device=self.dev)
        self.anchors = self.X.clone()
        n = self.X.shape[0]
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.U = torch.empty((3, n), **f64)          # u* then u'
        self.Xs = torch.empty((n, 3), **f64)         # X*
        self.F = torch.empty((3, n), **f64)          # tether forces
        self.ell = [torch.empty(g.point_count(), **f64) for g in self.grids]
        # One binning of X^n per component, shared by steps (a) and (e).
        self.binned = [None, None, None]

    def _components(self, fn):
        """fn(a) for the three components, concurrently when configured."""
        import torch

        if not self.concurrent:
            for a in range(3):
                fn(a)
            return
        main = torch.cuda.current_stream(self.dev)
        for a in range(3):
            self.streams[a].wait_stream(main)
            with torch.cuda.stream(self.streams[a]):
                fn(a)
        for a in range(3):
            main.wait_stream(self.streams[a])

    def _bin_and_interpolate(self, a):
        ops = self.comp_ops[a]
        self.binned[a] = ops.bin_points(self.X, self.grids[a], binned=self.binned[a])
        ops.interpolate_binned(self.velocity[a], self.binned[a], out=self.U[a])

    def _interpolate_vector(self, rebin: bool):
        if rebin:
            self._components(self._bin_and_interpolate)
        else:
            self._components(lambda a: self.comp_ops[a].interpolate_binned(
                self.velocity[a], self.binned[a], out=self.U[a]))

    def _spread_vector(self):
        self._components(lambda a: self.comp_ops[a].spread(
            self.Xs, self.F[a], self.grids[a], out=self.ell[a]))

    def step(self, events=None):
        """One reference step; `events` (optional) receives CUDA event pairs
        around (a), (d), (e) on the caller's stream."""
        import torch

        c = self.cfg

        def timed(key, fn):
            if events is None:
                fn()
                return
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            events.setdefault(key, []).append((e0, e1))

        timed("interpolate", lambda: self._interpolate_vector(rebin=True))      # (a)
        torch.add(self.X, self.U.t(), alpha=c.dt_s, out=self.Xs)                # (b)
        hookean_force(self.Xs, self.anchors, c.spring_constant, c.edge_cm, out=self.F)  # (c)
        timed("spread", self._spread_vector)                                    # (d)
        # X^n is unchanged since (a): its binning is reused.
        timed("interpolate", lambda: self._interpolate_vector(rebin=False))     # (e)
        self.X.add_(self.U.t(), alpha=c.dt_s)                                   # (f)

    @property
    def spread_result(self):
        return self.ell


# ---------------------------------------------------------------- reporting
def fnv1a(data, h: int = 14695981039346656037) -> int:
    """ib::bench::fnv1a (run.hpp:44-52), 64-bit FNV-1a over raw bytes
    (a numpy array or bytes; computed by libibcuda's ibc_fnv1a)."""
    import ctypes as C

    import numpy as np

    from . import _capi

    buf = np.ascontiguousarray(np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray))
                               else data)
    return int(_capi.load().ibc_fnv1a(buf.ctypes.data_as(C.c_void_p), buf.nbytes, h))


@dataclass
class TimingReport:
    """ib::bench::TimingReport (run.hpp:36-42); seconds are device times."""

    config: StepConfig
    interpolate_seconds: list = field(default_factory=list)
    spread_seconds: list = field(default_factory=list)
    final_positions: object = None
    physics_fingerprint: int = 0


def run_benchmark(cfg: StepConfig, device: int = 0, fingerprint: bool = True) -> TimingReport:
    """ib::bench::run_benchmark (run.hpp:59-128) on one GPU: cfg.steps steps,
    two interpolate_vector timings and one spread_vector timing per step
    (CUDA events), the final positions and the physics fingerprint (FNV-1a of
    the positions, then of each spread component, run.hpp:120-126)."""
    import torch

    loop = MacStepLoop(cfg, device)
    events: dict = {}
    for _ in range(cfg.steps):
        loop.step(events)
    torch.cuda.synchronize(device)
    rep = TimingReport(cfg)
    rep.interpolate_seconds = [a.elapsed_time(b) * 1e-3 for a, b in events.get("interpolate", [])]
    rep.spread_seconds = [a.elapsed_time(b) * 1e-3 for a, b in events.get("spread", [])]
    rep.final_positions = loop.X.cpu().numpy()
    if fingerprint:
        h = fnv1a(rep.final_positions)
        if cfg.steps > 0:
            for comp in loop.ell:
                h = fnv1a(comp.cpu().numpy(), h)
        rep.physics_fingerprint = h
    return rep


CSV_HEADER = ("algorithm,refinement,n_points,workers,sweep_width,operation,calls,mean_s,min_s,"
              "max_s,seed")  # report.hpp:16-18


def _csv_row(rep: TimingReport, op: str, secs) -> str:
    c = rep.config
    mean = sum(secs) / len(secs) if secs else 0.0
    mn, mx = (min(secs), max(secs)) if secs else (0.0, 0.0)
    return (f"{c.algorithm},{c.refinement},{c.point_count},{c.workers},{c.sweep_width},{op},"
            f"{len(secs)},{mean:.9e},{mn:.9e},{mx:.9e},{c.seed}")


def write_csv(reports, stream) -> None:
    """ib::bench::write_csv (report.hpp:60-66): header, then per report the
    interpolate row and the spread row."""
    stream.write(CSV_HEADER + "\n")
    for r in reports:
        stream.write(_csv_row(r, "interpolate", r.interpolate_seconds) + "\n")
        stream.write(_csv_row(r, "spread", r.spread_seconds) + "\n")
