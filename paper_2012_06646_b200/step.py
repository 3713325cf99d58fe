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

This is SURVEY.md 8(f) item 2 and the "MAC vector step" secondary figure of
8(d); the headline metric stays the scalar spread + interpolation pair.
"""
from __future__ import annotations

from dataclasses import dataclass

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

    def _interpolate_vector(self):
        self._components(lambda a: self.comp_ops[a].interpolate(
            self.velocity[a], self.X, self.grids[a], out=self.U[a]))

    def step(self):
        c = self.cfg
        self._interpolate_vector()                                        # (a)
        torch = __import__("torch")
        torch.add(self.X, self.U.t(), alpha=c.dt_s, out=self.Xs)          # (b)
        hookean_force(self.Xs, self.anchors, c.spring_constant, c.edge_cm, out=self.F)  # (c)
        self._components(lambda a: self.comp_ops[a].spread(               # (d)
            self.Xs, self.F[a], self.grids[a], out=self.ell[a]))
        self._interpolate_vector()                                        # (e)
        self.X.add_(self.U.t(), alpha=c.dt_s)                             # (f)

    @property
    def spread_result(self):
        return self.ell
