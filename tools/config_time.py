"""Dev: time + spot-check the BASELINE configs on one GPU.
usage: [IBC_DEV_PATH=auto|bank|pull|radix|walk] config_time.py [c1|c2|w128|w256|rbc|clustered|severe ...]"""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import oracle as O
from paper_2012_06646_b200 import ib, synth
from paper_2012_06646_b200.device import DeviceOperators

EDGE = 16e-4
def cfg(name):
    if name == "c1": N, pts = 64, synth.scatter_points(1 << 16, EDGE, 1)
    elif name == "c2": N, pts = 256, synth.scatter_points(1 << 20, EDGE, 1)
    elif name == "w128": N, pts = 128, synth.scatter_points(128 ** 3, EDGE, 1)
    elif name == "w256": N, pts = 256, synth.scatter_points(256 ** 3, EDGE, 1)
    elif name == "rbc": N = 256; pts = synth.rbc_points(EDGE, EDGE / N, 7)
    elif name == "clustered": N = 512; pts = synth.clustered_points(1 << 22, EDGE, 64, 8 * EDGE / 512, 5)
    elif name == "severe": N = 512; pts = synth.clustered_points(1 << 22, EDGE, 16, 4 * EDGE / 512, 5)
    return N, pts

ops = DeviceOperators(0)
ops.context.set_spread_path(os.environ.get("IBC_DEV_PATH", "auto"))
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for name in sys.argv[1:] or ["c1", "c2", "w128", "rbc", "clustered"]:
    N, pts = cfg(name)
    n = len(pts); h = EDGE / N
    g = ib.StaggeredGrid([N] * 3, h, [0.5, 0.5, 0.0], [True] * 3)
    xs = torch.tensor(synth.perturb(pts, 0.1 * h, 3), device="cuda")
    xn = torch.tensor(pts, device="cuda")
    G = torch.tensor(synth.uniform_pm1(n, 2), device="cuda")
    e = torch.tensor(synth.uniform_pm1(N ** 3, 4), device="cuda")
    l = torch.empty(N ** 3, dtype=torch.float64, device="cuda"); E = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        ops.spread(xs, G, g, out=l); ops.interpolate(e, xn, g, out=E)
    torch.cuda.synchronize()
    ts, tsp, tin = [], [], []
    for it in range(10):
        flush.fill_(it)
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(); ops.spread(xs, G, g, out=l); b.record(); ops.interpolate(e, xn, g, out=E); c.record()
        torch.cuda.synchronize()
        tsp.append(a.elapsed_time(b)); tin.append(b.elapsed_time(c))
    sp, it_ = np.median(tsp), np.median(tin)
    ops.context.set_profiling(True); ops.context.reset_profile()
    for it in range(3):
        flush.fill_(it); ops.spread(xs, G, g, out=l); ops.interpolate(e, xn, g, out=E)
    pr = ops.context.profile(); ops.context.set_profiling(False)
    print("   ", {k: round(v / 3 * 1e3, 1) for k, v in pr.items() if k.endswith("_ms")}, flush=True)
    alg = 64 * n + 16 * N ** 3
    # spot check against the oracle on a 20k-point subsample
    k = min(n, 20000)
    og = O.make_grid([N] * 3, h, [0.5, 0.5, 0.0], [1, 1, 1])
    sub = slice(0, k)
    ls = torch.empty(N ** 3, dtype=torch.float64, device="cuda")
    ops.spread(xs[sub].contiguous(), G[sub].contiguous(), g, out=ls)
    dev_s = O.max_rel_deviation(ls.cpu().numpy(), O.spread_serial(og, xs[sub].cpu().numpy(), G[sub].cpu().numpy()))
    dev_i = O.max_rel_deviation(E[sub].cpu().numpy(), O.interpolate(og, e.cpu().numpy(), xn[sub].cpu().numpy()))
    print(f"{name:10s} n={n:9d} N={N}: spread {sp*1e3:8.1f} us interp {it_*1e3:8.1f} us -> "
          f"{n/(sp+it_)*1e3:.3e} pts/s, step roofline {alg/((sp+it_)*1e-3)/6.5459e12:.3f}; dev {dev_s:.1e} {dev_i:.1e}", flush=True)
