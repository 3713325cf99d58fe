"""Dev probe: clock64 timeline of one spread / interp z-sweep CTA at config 2."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2012_06646_b200 import ib, _capi
from paper_2012_06646_b200.device import DeviceOperators
lib = _capi.load()
lib.ibc_debug_zsweep_trace.argtypes = [C.c_int, C.c_void_p]
n, N, edge = 1 << 20, 256, 16e-4
h = edge / N
g = ib.StaggeredGrid([N]*3, h, [0.5, 0.5, 0.0], [True]*3)
rng = np.random.default_rng(1)
x = torch.tensor(rng.uniform(0, edge, (n, 3)), device="cuda")
G = torch.tensor(rng.uniform(-1, 1, n), device="cuda")
e = torch.tensor(rng.uniform(-1, 1, N**3), device="cuda")
ops = DeviceOperators(0)
l = ops.spread(x, G, g); E = ops.interpolate(e, x, g); torch.cuda.synchronize()
for blk in (0, 300, 700):
    lib.ibc_debug_zsweep_trace(blk, None)
    ops.spread(x, G, g, out=l); ops.interpolate(e, x, g, out=E); torch.cuda.synchronize()
    buf = np.zeros(2 * 64 * 8, np.int64)
    lib.ibc_debug_zsweep_trace(-1, buf.ctypes.data)
    buf = buf.reshape(2, 64, 8)
    for which, name in ((0, "spread"), (1, "interp")):
        t = buf[which]
        steps = [i for i in range(64) if t[i, 0]]
        if not steps: continue
        t0 = t[steps[0], 0]
        print(f"block {blk} {name}: steps={len(steps)} total={t[steps[-1]].max() - t0} cycles")
        for i in steps[:6] + steps[-2:]:
            row = t[i]
            print("  step", i, [int(v - row[0]) if v else None for v in row])
