import sys; sys.path.insert(0, '.')

import numpy as np, torch
import oracle as O
from paper_2012_06646_b200 import ib
rng = np.random.default_rng(21)
K = ib.CosineKernel()
cases = [([40, 36, 24], [True] * 3, 6000), ([33, 20, 18], [False, True, False], 4000),
         ([24, 16], [True, False], 3000)]
for ext, per, n in cases:
    g = ib.StaggeredGrid(ext, 0.5, [0.5] * len(ext), per)
    L = np.array(ext) * 0.5
    pts = rng.uniform(-0.2 * L, 1.2 * L, (n, len(ext)))
    pts[: n // 3] = pts[0] + rng.normal(0, 0.3, (n // 3, len(ext)))  # a cluster
    vals = rng.uniform(-1, 1, n)
    ws = ib.SpreadWorkspace(n, g)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    og = O.make_grid(g.extents, g.spacing(), g.staggerings, g.periodic, g.origin)
    want, keys, perm, runs = O.spread_fused(og, pts, vals)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm), ext
    assert ws.run_count == len(runs)
    assert O.max_rel_deviation(got.values, want) <= 1e-12, ext
    again = ib.spread_fused(pts, vals, g, K, ws, 8)
    assert np.array_equal(again.values, got.values)  # deterministic
print("ok")
