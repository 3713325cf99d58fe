"""Dev timing probe: per-kernel-class device times at BASELINE config 2."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2012_06646_b200 import ib
from paper_2012_06646_b200.device import DeviceOperators

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
N = int(sys.argv[2]) if len(sys.argv) > 2 else 256
edge = 16e-4; h = edge / N
g = ib.StaggeredGrid([N]*3, h, [0.5, 0.5, 0.0], [True]*3)
rng = np.random.default_rng(1)
xn = torch.tensor(rng.uniform(0, edge, (n, 3)), device="cuda")
xs = (xn + torch.tensor(rng.uniform(-0.1*h, 0.1*h, (n, 3)), device="cuda")).contiguous()
G = torch.tensor(rng.uniform(-1, 1, n), device="cuda")
e = torch.tensor(rng.uniform(-1, 1, N**3), device="cuda")
ops = DeviceOperators(0)
l = torch.empty(N**3, dtype=torch.float64, device="cuda"); E = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    ops.spread(xs, G, g, out=l); ops.interpolate(e, xn, g, out=E)
torch.cuda.synchronize()
flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ts = []
for it in range(20):
    flush.fill_(it)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); ops.spread(xs, G, g, out=l); ops.interpolate(e, xn, g, out=E); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ts = np.array(ts)
alg = 64 * n + 16 * N**3
print(f"n={n} N={N} step median {np.median(ts)*1e3:.1f} us min {ts.min()*1e3:.1f} us -> {n/np.median(ts)*1e3:.3e} pts/s, "
      f"{alg/np.median(ts)/1e6:.0f} GB/s alg")
ops.context.set_profiling(True); ops.context.reset_profile()
for it in range(10):
    flush.fill_(it)
    ops.spread(xs, G, g, out=l); ops.interpolate(e, xn, g, out=E)
p = ops.context.profile()
print({k: (round(v/10*1e3, 1) if k.endswith('ms') else v) for k, v in p.items()}, "(us per step)")
