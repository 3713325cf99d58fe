import sys, numpy as np
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O
from paper_2012_06646_b200 import ib
z = np.load("tests/golden/golden_small.npz")
for c in range(int(z["ncases"][0])):
    p = f"c{c}_"
    ext = list(z[p+"ext"])
    if len(ext) < 2: continue
    g = ib.StaggeredGrid(ext, float(z[p+"h"][0]), list(z[p+"alpha"]), [bool(v) for v in z[p+"per"]])
    pts, vals = z[p+"pts"], z[p+"vals"]
    ws = ib.SpreadWorkspace(len(vals), g)
    got = ib.spread_fused(pts, vals, g, ib.CosineKernel(), ws, 4)
    d = O.max_rel_deviation(got.values, z[p+"spread"])
    print(c, ext, list(z[p+"per"]), len(vals), d)
    if d > 1e-12:
        diff = np.abs(got.values - z[p+"spread"]).reshape(ext[::-1])
        print("bad at", np.argwhere(diff > 1e-9)[:10].tolist())
        break
