import sys, numpy as np
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O
from paper_2012_06646_b200 import ib
np.set_printoptions(linewidth=200, precision=3, suppress=True)
z = np.load("tests/golden/golden_small.npz")
for c in [1, 2, 4, 5]:
    p = f"c{c}_"
    ext = list(z[p+"ext"])
    g = ib.StaggeredGrid(ext, float(z[p+"h"][0]), list(z[p+"alpha"]), [bool(v) for v in z[p+"per"]])
    pts, vals = z[p+"pts"], z[p+"vals"]
    ws = ib.SpreadWorkspace(len(vals), g)
    got = ib.spread_fused(pts, vals, g, ib.CosineKernel(), ws, 4)
    want = z[p+"spread"]
    print("case", c, ext, z[p+"per"], "dev", O.max_rel_deviation(got.values, want))
    if len(ext) == 2:
        print((got.values - want).reshape(ext[::-1]))
    # single-point probes
    for i in range(3):
        g1 = ib.spread_fused(pts[i:i+1], vals[i:i+1], g, ib.CosineKernel(), ib.SpreadWorkspace(1, g), 1)
        og = O.make_grid(ext, float(z[p+"h"][0]), list(z[p+"alpha"]), list(z[p+"per"]))
        w1 = O.spread_serial(og, pts[i:i+1], vals[i:i+1]) if hasattr(O, "spread_serial") else O.spread_fused(og, pts[i:i+1], vals[i:i+1])[0]
        print("  single", i, pts[i], O.max_rel_deviation(g1.values, w1))
