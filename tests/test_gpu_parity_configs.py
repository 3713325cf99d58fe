"""Parity on what the bench and the BASELINE configs actually run (B200).

* The TMA-fed interpolation gather (3-D, nx % 16 == 0 -- every BASELINE
  config) and the bank-mode spread on grids with a closed x, y or z axis:
  ghost home cells -1 / n, points within two cells of the walls, the TMA
  out-of-bounds zero fill and the off-grid x weights
  (interpolate.hpp:42-52 skips off < 0; support_window.hpp:22-42).
* Config 2 interpolation at full size, W-128 full-array, W-512 sampled (whole
  planes of the spread, 2^20 sampled interpolation outputs), C-severe
  full-array.

Bar as everywhere: keys / permutations / run counts bit-exact, values within
max_rel_deviation <= 1e-12 (FP64, inc/bench/verify.hpp:36-45).
"""
import numpy as np
import pytest

import oracle as O
from paper_2012_06646_b200 import ib

pytestmark = pytest.mark.gpu

K = ib.CosineKernel()
TOL = 1e-12
EDGE = 16e-4  # SURVEY 8(d) domain, cm


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def og(g):
    return O.make_grid(g.extents, g.spacing(), g.staggerings, g.periodic, g.origin)


def wall_points(g, n, rng, band_frac=0.4):
    """Points whose home cells cover the extended range [-1, n] of every closed
    axis: a share of them within two cells of each wall (home cells -1, 0, 1
    and n-2 .. n), the rest uniform; periodic axes span three periods."""
    h = g.spacing()
    pts = np.empty((n, g.dim))
    for a in range(g.dim):
        o, al, e = g.origin[a], g.staggerings[a], g.extents[a]
        if g.is_periodic(a):
            L = g.axis_length(a)
            pts[:, a] = o + rng.uniform(-L, 2 * L, n)
            continue
        # home c = ceil((x - o)/h - alpha) in [-1, e]  <=>  x in (o + h(alpha-2), o + h(alpha+e)]
        lo, hi = o + h * (al - 2.0) + 1e-9 * h, o + h * (al + e)
        x = rng.uniform(lo, hi, n)
        band = rng.random(n) < band_frac
        side = rng.random(n) < 0.5
        nb = int(band.sum())
        x[band & side] = rng.uniform(lo, lo + 3.0 * h, int((band & side).sum()))
        x[band & ~side] = rng.uniform(hi - 3.0 * h, hi, nb - int((band & side).sum()))
        pts[:, a] = x
    return pts


def _check_both(g, pts, vals, field, keys_too=True):
    ws = ib.SpreadWorkspace(len(vals), g)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    o = og(g)
    if keys_too:
        want, keys, perm, run_keys = O.spread_fused(o, pts, vals)
        assert np.array_equal(ws.keys, keys)
        assert np.array_equal(ws.perm, perm)
        assert ws.run_count == run_keys.size
    else:
        want = O.spread_serial(o, pts, vals)
    assert O.max_rel_deviation(got.values, want) <= TOL
    E = ib.interpolate(ib.GridField(g, field), pts, K, 8)
    assert O.max_rel_deviation(E, O.interpolate(o, field, pts)) <= TOL
    return got.values, E


CLOSED = {"x": (False, True, True), "y": (True, False, True), "z": (True, True, False),
          "xyz": (False, False, False), "xz": (False, True, False)}


@pytest.mark.parametrize("nx", [64, 128, 256])
@pytest.mark.parametrize("closed", sorted(CLOSED))
def test_tma_gather_and_bank_spread_with_closed_axes(nx, closed):
    rng = np.random.default_rng(1000 + nx + len(closed) * 7 + ord(closed[0]))
    ny, nz = (40, 36) if nx == 256 else (nx // 2 + 8, nx // 2 - 4)
    g = ib.StaggeredGrid([nx, ny, nz], 0.125, [0.5, 0.25, 0.0], list(CLOSED[closed]),
                         [0.3, -1.1, 0.7])
    n = 60000 if nx == 256 else 30000
    pts = wall_points(g, n, rng)
    vals = rng.uniform(-1, 1, n)
    field = rng.uniform(-1, 1, g.point_count())
    _check_both(g, pts, vals, field)


def test_tma_gather_closed_cube_every_ghost_row():
    # A closed 128^3 cube at config-2 density plus one point homed in every
    # ghost row (cy, cz) in {-1, n} x {-1, n} at x = -1, 0, n-1, n.
    rng = np.random.default_rng(77)
    N = 128
    g = ib.StaggeredGrid([N] * 3, EDGE / N, [0.5, 0.5, 0.0], [False] * 3)
    h = g.spacing()
    pts = [wall_points(g, 1 << 17, rng, band_frac=0.25)]
    for cx in (-1, 0, N - 1, N):
        for cy in (-1, 0, N - 1, N):
            for cz in (-1, 0, N - 1, N):
                c = np.array([cx, cy, cz], float)
                u = rng.uniform(0.05, 0.95, (3, 3))  # x = h (c + alpha - u)
                pts.append(h * (c + np.array([0.5, 0.5, 0.0]) - u))
    pts = np.concatenate(pts)
    vals = rng.uniform(-1, 1, len(pts))
    field = rng.uniform(-1, 1, g.point_count())
    assert O.home_cells(og(g), pts).min() == -1 and O.home_cells(og(g), pts).max() == N
    _check_both(g, pts, vals, field)


@pytest.mark.slow
def test_config2_interpolation_full_size():
    # BASELINE config 2 interpolation at X^n (2^20 points, 256^3, field seed 4)
    n, N = 1 << 20, 256
    g = ib.StaggeredGrid([N] * 3, EDGE / N, [0.5, 0.5, 0.0], [True] * 3)
    xn = O.scatter_points(n, EDGE, 1)
    e = 2.0 * O.scatter_points(N ** 3 // 3 + 1, 1.0, 4).reshape(-1)[: N ** 3] - 1.0
    E = ib.interpolate(ib.GridField(g, e), xn, K, 8)
    assert O.max_rel_deviation(E, O.interpolate(og(g), e, xn)) <= TOL
    # the perturbed X* of the bench step as well (a different sort)
    xs = xn + np.random.default_rng(3).uniform(-0.1, 0.1, xn.shape) * g.spacing()
    Es = ib.interpolate(ib.GridField(g, e), xs, K, 8)
    assert O.max_rel_deviation(Es, O.interpolate(og(g), e, xs)) <= TOL


@pytest.mark.slow
def test_weak_scaling_w128_full_array():
    # BASELINE config 3 at one GPU: 1 point per cell, 128^3 (2,097,152 points)
    N = 128
    g = ib.StaggeredGrid([N] * 3, EDGE / N, [0.5, 0.5, 0.0], [True] * 3)
    pts = O.scatter_points(N ** 3, EDGE, 1)
    rng = np.random.default_rng(41)
    vals = rng.uniform(-1, 1, N ** 3)
    field = rng.uniform(-1, 1, N ** 3)
    ws = ib.SpreadWorkspace(N ** 3, g)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    keys, perm, run_keys = O.prepare_keys(og(g), pts)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert ws.run_count == run_keys.size == 1326117
    assert O.max_rel_deviation(got.values, O.spread_serial(og(g), pts, vals)) <= TOL
    E = ib.interpolate(ib.GridField(g, field), pts, K, 8)
    assert O.max_rel_deviation(E, O.interpolate(og(g), field, pts)) <= TOL


@pytest.mark.slow
def test_weak_scaling_w512_sampled():
    """BASELINE config 3 at its largest level: 512^3 grid, 512^3 points
    (134 M), device-resident.  Sampled parity: keys and
    permutation in full; the spread on whole target planes -- one block
    across the periodic z seam, one interior -- against the oracle over every
    point that reaches them; 2^20 sampled interpolation outputs."""
    import torch

    from paper_2012_06646_b200.device import DeviceOperators

    N = 512
    n = N ** 3
    g = ib.StaggeredGrid([N] * 3, EDGE / N, [0.5, 0.5, 0.0], [True] * 3)
    o = og(g)
    pts = O.scatter_points(n, EDGE, 1)
    rng = np.random.default_rng(43)
    vals = rng.uniform(-1, 1, n)
    ops = DeviceOperators(0)
    dp = torch.from_numpy(pts).cuda()
    dv = torch.from_numpy(vals).cuda()
    ws = ops.workspace(n, g)
    ell = ops.spread(dp, dv, g, workspace=ws)
    torch.cuda.synchronize()
    del dv
    keys, perm, _ = O.prepare_keys(o, pts)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    del keys, perm
    cz = O.home_cells(o, pts)[:, 2]
    for planes in ([N - 2, N - 1, 0, 1], [200, 201, 202, 203]):
        # target plane t receives from home planes t-1 .. t+2 (shifts -2..1)
        reach = set()
        for t in planes:
            reach.update(((t + d) % N) for d in (-1, 0, 1, 2))
        sel = np.isin(cz, np.array(sorted(reach)))
        want = O.spread_serial(o, pts[sel], vals[sel]).reshape(N, N, N)[planes]
        got = ell.view(N, N, N)[planes].cpu().numpy()
        assert O.max_rel_deviation(got, want) <= TOL, planes
        del want
    del ell
    field_np = rng.uniform(-1, 1, n)
    E = ops.interpolate(torch.from_numpy(field_np).cuda(), dp, g)
    sample = rng.choice(n, 1 << 20, replace=False)
    want = O.interpolate(o, field_np, pts[sample])
    assert O.max_rel_deviation(E[torch.from_numpy(sample).cuda()].cpu().numpy(), want) <= TOL


@pytest.mark.slow
def test_config_clustered_severe_full_array():
    # SURVEY 8(d) config C, severe: 2^22 points in 16 clusters of sigma = 4h,
    # 512^3 (max run ~300 points per cell: the long bank lists)
    from paper_2012_06646_b200 import synth

    N = 512
    pts = synth.clustered_points(1 << 22, EDGE, 16, 4 * EDGE / N, 5)
    g = ib.StaggeredGrid([N] * 3, EDGE / N, [0.5, 0.5, 0.0], [True] * 3)
    rng = np.random.default_rng(47)
    vals = rng.uniform(-1, 1, len(pts))
    field = rng.uniform(-1, 1, g.point_count())
    _check_both(g, pts, vals, field)
