"""Run every golden case through spread_fused one by one (debug helper)."""
import sys, subprocess, numpy as np
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
z = np.load("tests/golden/golden_small.npz")
cases = sorted({k.split("_")[0] for k in z.files if k.startswith("c")}, key=lambda s: int(s[1:]))
if len(sys.argv) > 1:
    import oracle as O
    from paper_2012_06646_b200 import ib
    p = sys.argv[1] + "_"
    ext = list(z[p + "ext"])
    g = ib.StaggeredGrid(ext, float(z[p + "h"][0]), list(z[p + "alpha"]), [bool(v) for v in z[p + "per"]])
    pts, vals = z[p + "pts"], z[p + "vals"]
    got = ib.spread_fused(pts, vals, g, ib.CosineKernel(), ib.SpreadWorkspace(len(vals), g), 4)
    print("ok", O.max_rel_deviation(got.values, z[p + "spread"]))
    sys.exit(0)
for c in cases:
    r = subprocess.run([sys.executable, __file__, c], capture_output=True, text=True)
    p = c + "_"
    print(c, list(z[p + "ext"]), list(z[p + "per"]), len(z[p + "vals"]), r.stdout.strip()[-60:] or r.stderr.strip()[-120:])
