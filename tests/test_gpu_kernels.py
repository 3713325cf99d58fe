"""Every delta kernel the device takes, against the reference (B200).

The reference's operators are templates over any `Kernel` (kernel.hpp:16-21).
The device takes the kernels of `ibc_kernel`: the reference's CosineKernel,
Peskin's 4-point kernel (both on the fast paths -- bank / pull sweeps, TMA
gather -- through their per-axis weight pair), the odd-support 3-point
kernel of Roma, Peskin & Berger and the 2-point hat (generic radix-sorted
tiles).  Golden vectors: tests/golden/golden_kernels.npz, made by the
reference headers instantiated with those kernels (make_golden_kernels.py).
Bar: keys / perm / run keys bit-exact, values max_rel_deviation <= 1e-12.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2012_06646_b200 import ib

GOLD = Path(__file__).resolve().parent / "golden"
TOL = 1e-12
KERNEL_OF = {0: ib.CosineKernel(), 1: ib.Peskin4Kernel(), 2: ib.Roma3Kernel(), 3: ib.Linear2Kernel()}


def og(g):
    return O.make_grid(g.extents, g.spacing(), g.staggerings, g.periodic, g.origin)


def test_python_kernels_match_oracle_phi():
    # CPU: the host-side phi of every kernel class equals the oracle's
    for k, kern in KERNEL_OF.items():
        assert kern.support() == O.lib().or_kernel_support(k)
        for r in np.linspace(-2.6, 2.6, 113):
            assert kern.phi(r) == pytest.approx(O.kernel_phi(k, r), abs=1e-16), (k, r)


def test_unknown_kernel_type_is_rejected():
    # CPU: a caller's own Kernel type is not silently mapped onto a device kernel
    class MyKernel:
        code = 0  # even one that claims a device id

        def phi(self, r):
            return 0.0

        def support(self):
            return 4

        def radius(self):
            return 2.0

    with pytest.raises(ib.InvalidArgument):
        ib._kernel_code(MyKernel())
    assert ib._kernel_code(ib.Peskin4Kernel()) == 1 and ib._kernel_code(ib.Roma3Kernel) == 2


@pytest.fixture()
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
def test_golden_kernels_bit_exact_keys_and_values(_cuda):
    z = np.load(GOLD / "golden_kernels.npz")
    for c in range(int(z["ncases"][0])):
        p = f"c{c}_"
        kern = KERNEL_OF[int(z[p + "kernel"][0])]
        g = ib.StaggeredGrid(list(z[p + "ext"]), float(z[p + "h"][0]), list(z[p + "alpha"]),
                             [bool(v) for v in z[p + "per"]], list(z[p + "origin"]))
        pts, vals = z[p + "pts"], z[p + "vals"]
        ws = ib.SpreadWorkspace(len(vals), g)
        got = ib.spread_fused(pts, vals, g, kern, ws, 2)
        assert np.array_equal(ws.keys, z[p + "keys"]), c
        assert np.array_equal(ws.perm, z[p + "perm"]), c
        assert np.array_equal(ws.run_keys, z[p + "run_keys"]), c
        assert O.max_rel_deviation(got.values, z[p + "spread"]) <= TOL, c
        assert O.max_rel_deviation(got.values, z[p + "serial"]) <= TOL, c
        e = ib.interpolate(ib.GridField(g, z[p + "field"]), pts, kern, 2)
        assert O.max_rel_deviation(e, z[p + "interp"]) <= TOL, c


def _rand_points(g, n, rng):
    pts = np.empty((n, g.dim))
    for a in range(g.dim):
        L = g.axis_length(a)
        o = g.origin[a]
        pts[:, a] = o + (rng.uniform(-L, 2 * L, n) if g.is_periodic(a) else rng.uniform(0, L, n))
    return pts


@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 1, 2, 3])
@pytest.mark.parametrize("per", [(True, True, True), (False, True, False)])
@pytest.mark.parametrize("path", ["auto", "bank", "pull", "radix"])
def test_kernels_on_3d_grids_every_spread_path(_cuda, k, per, path):
    # 64 x 48 x 40: the TMA gather and the sweeps for the 4-point kernels,
    # the generic tiles for supports 3 and 2; dense enough for pull mode.
    rng = np.random.default_rng(100 + 10 * k + sum(per))
    kern = KERNEL_OF[k]
    g = ib.StaggeredGrid([64, 48, 40], 0.25, [0.5, 0.25, 0.0], list(per), [0.1, -0.3, 0.2])
    n = 60000
    pts = _rand_points(g, n, rng)
    vals = rng.uniform(-1, 1, n)
    ctx = ib.Context(0)
    ctx.set_spread_path(path)
    ws = ib.SpreadWorkspace(n, g, context=ctx)
    got = ib.spread_fused(pts, vals, g, kern, ws, 8)
    want, keys, perm, run_keys = O.spread_fused(og(g), pts, vals, kernel=k)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert ws.run_count == run_keys.size
    assert O.max_rel_deviation(got.values, want) <= TOL
    e = rng.uniform(-1, 1, g.point_count())
    E = ib.interpolate(ib.GridField(g, e), pts, kern, 8)
    assert O.max_rel_deviation(E, O.interpolate(og(g), e, pts, kernel=k)) <= TOL


@pytest.mark.gpu
def test_peskin4_config2_full_size(_cuda):
    # BASELINE names "the 4-point Peskin delta kernel": config 2 with it
    n, N, edge = 1 << 20, 256, 16e-4
    g = ib.StaggeredGrid([N] * 3, edge / N, [0.5, 0.5, 0.0], [True] * 3)
    pts = O.scatter_points(n, edge, 1)
    vals = 2.0 * O.scatter_points(n, 1.0, 2)[:, 0] - 1.0
    ws = ib.SpreadWorkspace(n, g)
    got = ib.spread_fused(pts, vals, g, ib.Peskin4Kernel(), ws, 8)
    keys, perm, run_keys = O.prepare_keys(og(g), pts, kernel=1)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert O.max_rel_deviation(got.values, O.spread_serial(og(g), pts, vals, kernel=1)) <= TOL
    e = np.random.default_rng(4).uniform(-1, 1, N ** 3)
    E = ib.interpolate(ib.GridField(g, e), pts, ib.Peskin4Kernel(), 8)
    assert O.max_rel_deviation(E, O.interpolate(og(g), e, pts, kernel=1)) <= TOL


@pytest.mark.gpu
def test_operation_counts_follow_support(_cuda):
    # stats::add_delta_evaluations adds n * s^d (stats.hpp:23-25, spread.hpp:158)
    g = ib.StaggeredGrid([8, 8, 8], 0.5, [0.0] * 3, [True] * 3)
    pts = _rand_points(g, 100, np.random.default_rng(1))
    for k, kern in KERNEL_OF.items():
        ib.stats.reset_delta_evaluations()
        ib.spread_serial(pts, np.ones(100), g, kern)
        ib.interpolate(ib.GridField(g), pts, kern)
        assert ib.stats.delta_evaluations() == 2 * 100 * kern.support() ** 3
