import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2012_06646_b200 import ib, synth
from paper_2012_06646_b200.device import DeviceOperators, capture_graph
N, n, EDGE = 256, 1 << 20, 16e-4; h = EDGE / N
g = ib.StaggeredGrid([N] * 3, h, [0.5, 0.5, 0.0], [True] * 3)
pts = synth.scatter_points(n, EDGE, 1)
ops = DeviceOperators(0)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for dt in (torch.float64, torch.float32):
    xs = torch.tensor(synth.perturb(pts, 0.1 * h, 3), device="cuda").to(dt)
    xn = torch.tensor(pts, device="cuda").to(dt)
    G = torch.tensor(synth.uniform_pm1(n, 2), device="cuda").to(dt)
    e = torch.tensor(synth.uniform_pm1(N ** 3, 4), device="cuda").to(dt)
    l = torch.empty(N ** 3, dtype=dt, device="cuda"); E = torch.empty(n, dtype=dt, device="cuda")
    fn = lambda: (ops.spread(xs, G, g, out=l), ops.interpolate(e, xn, g, out=E))
    for _ in range(3): fn()
    gr = capture_graph(fn)
    ts = []
    for it in range(20):
        flush.fill_(it)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    print(dt, f"median {np.median(ts):.1f} us -> {n / np.median(ts) * 1e6:.3e} pts/s")
