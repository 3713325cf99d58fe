"""Every spread path against the oracle: bank mode, pull mode and the radix
sort path, forced per context (ibc_context_set_spread_path)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2012_06646_b200 import ib

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
K = ib.CosineKernel()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("path", ["pull", "bank", "radix", "auto"])
def test_spread_paths_match_oracle(path):
    rng = np.random.default_rng(21)
    ctx = ib.Context(0)
    ctx.set_spread_path(path)
    cases = [([40, 36, 24], [True] * 3, 6000), ([33, 20, 18], [False, True, False], 4000),
             ([24, 16], [True, False], 3000), ([64, 48, 40], [True] * 3, 20000)]
    for ext, per, n in cases:
        g = ib.StaggeredGrid(ext, 0.5, [0.5] * len(ext), per)
        L = np.array(ext) * 0.5
        lo = np.where(per, -0.2 * L, 0.0)   # closed axes: inside the domain (the
        hi = np.where(per, 1.2 * L, L)      # reference's tests' contract)
        pts = rng.uniform(lo, hi, (n, len(ext)))
        pts[: n // 3] = np.clip(pts[0] + rng.normal(0, 0.3, (n // 3, len(ext))), lo, hi - 1e-9)
        vals = rng.uniform(-1, 1, n)
        ws = ib.SpreadWorkspace(n, g, context=ctx)
        got = ib.spread_fused(pts, vals, g, K, ws, 8)
        og = O.make_grid(g.extents, g.spacing(), g.staggerings, g.periodic, g.origin)
        want, keys, perm, runs = O.spread_fused(og, pts, vals)
        assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm), ext
        assert ws.run_count == len(runs)
        assert O.max_rel_deviation(got.values, want) <= 1e-12, ext
        again = ib.spread_fused(pts, vals, g, K, ws, 8)
        assert np.array_equal(again.values, got.values)  # deterministic
    ctx.close()


def test_spread_path_rejects_unknown():
    with pytest.raises(ib.InvalidArgument):
        ib.default_context().set_spread_path("fastest")


FAR = r'''
import numpy as np, torch
import oracle as O
from paper_2012_06646_b200 import ib
rng = np.random.default_rng(22)
K = ib.CosineKernel()
g = ib.StaggeredGrid([30, 24, 20], 0.5, [0.5, 0.5, 0.0], [False, True, False])
L = np.array(g.extents) * 0.5
inside = rng.uniform([0, -3, 0], L + [0, 3, 0], (3000, 3))
far = rng.uniform([0, 0, 0], L, (500, 3))
far[:, 0] += np.where(rng.random(500) < 0.5, -1, 1) * (L[0] + 4.0)  # > 4 cells outside x
pts = np.concatenate([inside, far])
vals = rng.uniform(-1, 1, len(pts))
got = ib.spread_fused(pts, vals, g, K, ib.SpreadWorkspace(len(pts), g), 8)
og = O.make_grid(g.extents, g.spacing(), g.staggerings, g.periodic, g.origin)
assert O.max_rel_deviation(got.values, O.spread_serial(og, inside, vals[:3000])) <= 1e-12
e = rng.uniform(-1, 1, g.point_count())
E = ib.interpolate(ib.GridField(g, e), pts, K)
assert O.max_rel_deviation(E[:3000], O.interpolate(og, e, inside)) <= 1e-12
assert not np.any(E[3000:])
print("ok")
'''


def test_points_far_outside_a_closed_axis_are_ignored():
    """Points homed > 2 cells outside a closed axis reach no grid point (the
    reference drops their targets as invalid offsets); they must not disturb
    the others -- their keys alias other rows, so they are bucketed apart."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    e = dict(os.environ, PYTHONPATH=str(ROOT))
    out = subprocess.run([sys.executable, "-c", FAR], cwd=ROOT, env=e, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stdout + out.stderr
