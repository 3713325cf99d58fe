import sys; sys.path.insert(0, '.')

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
