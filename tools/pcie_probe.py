"""PCIe floor of the end-to-end config-2 step: the box's pinned-memory copy
bandwidth (H2D alone, D2H alone, both directions at once, in the 8 MiB pieces
the library uses) next to the C-ABI host-buffer calls (ibc_spread,
ibc_interpolate) alone and issued concurrently from two threads.
usage: python tools/pcie_probe.py [reps]"""
import ctypes as C
import statistics
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2012_06646_b200 import _capi, ib, synth

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
N, n, EDGE = 256, 1 << 20, 16e-4
h = EDGE / N
H2D, D2H = 24 * n + 8 * n + 8 * N ** 3 + 24 * n, 8 * N ** 3 + 8 * n  # bytes per step
PIECE = 8 << 20


def med(f):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


hsrc = torch.empty(H2D, dtype=torch.uint8).pin_memory()
hdst = torch.empty(D2H, dtype=torch.uint8).pin_memory()
dsrc = torch.empty(D2H, dtype=torch.uint8, device="cuda")
ddst = torch.empty(H2D, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def h2d():
    with torch.cuda.stream(s1):
        for o in range(0, H2D, PIECE):
            ddst[o:o + PIECE].copy_(hsrc[o:o + PIECE], non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        for o in range(0, D2H, PIECE):
            hdst[o:o + PIECE].copy_(dsrc[o:o + PIECE], non_blocking=True)


def both():
    h2d()
    d2h()


t_h, t_d, t_b = med(h2d), med(d2h), med(both)
print(f"H2D {H2D / 1e6:.0f} MB alone: {t_h * 1e3:.2f} ms = {H2D / t_h / 1e9:.1f} GB/s")
print(f"D2H {D2H / 1e6:.0f} MB alone: {t_d * 1e3:.2f} ms = {D2H / t_d / 1e9:.1f} GB/s")
print(f"both directions at once: {t_b * 1e3:.2f} ms  (floor of a step's copies)")

g = ib.StaggeredGrid([N] * 3, h, [0.5, 0.5, 0.0], [True] * 3)
pts = synth.scatter_points(n, EDGE, 1)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hx_s, hx_n = pin(synth.perturb(pts, 0.1 * h, 3)), pin(pts)
hg, hf = pin(synth.uniform_pm1(n, 2)), pin(synth.uniform_pm1(N ** 3, 4))
h_ell = torch.empty(N ** 3, dtype=torch.float64).pin_memory()
h_E = torch.empty(n, dtype=torch.float64).pin_memory()
lib = _capi.load()
ctx = ib.default_context(0)
ws = ib.SpreadWorkspace(n, g, context=ctx)
vp = lambda t: C.c_void_p(t.data_ptr())


def spread_call():
    _capi.check(lib.ibc_spread(ctx.handle, C.byref(g.c_grid), _capi.IBC_KERNEL_COSINE4,
                               _capi.IBC_SPREAD_FUSED, vp(hx_s), vp(hg), n, n, 0, ws.handle, 0,
                               vp(h_ell)))


def interp_call():
    _capi.check(lib.ibc_interpolate(ctx.handle, C.byref(g.c_grid), _capi.IBC_KERNEL_COSINE4,
                                    vp(hf), vp(hx_n), n, 0, vp(h_E)))


pool = ThreadPoolExecutor(max_workers=1)


def pair():
    fut = pool.submit(interp_call)
    spread_call()
    fut.result()


def pair_seq():
    spread_call()
    interp_call()


t_s, t_i, t_p, t_q = med(spread_call), med(interp_call), med(pair), med(pair_seq)
print(f"ibc_spread alone {t_s * 1e3:.2f} ms, ibc_interpolate alone {t_i * 1e3:.2f} ms, "
      f"back to back {t_q * 1e3:.2f} ms, two threads {t_p * 1e3:.2f} ms = {n / t_p:.3e} points/s "
      f"({t_b / t_p:.0%} of the copy floor)")



def pair_timeline():
    t0 = time.perf_counter()
    done = {}

    def ti():
        interp_call()
        done["interp"] = time.perf_counter() - t0
    fut = pool.submit(ti)
    spread_call()
    done["spread"] = time.perf_counter() - t0
    fut.result()
    return done


pair_timeline()
tl = [pair_timeline() for _ in range(reps)]
print("two threads, call returns after: spread " +
      f"{statistics.median(d['spread'] for d in tl) * 1e3:.2f} ms, interpolation "
      f"{statistics.median(d['interp'] for d in tl) * 1e3:.2f} ms")


props = torch.cuda.get_device_properties(0)
bus = f"{getattr(props, 'pci_domain_id', 0):04x}:{getattr(props, 'pci_bus_id', 0):02x}:{getattr(props, 'pci_device_id', 0):02x}.0"
try:
    node = Path(f"/sys/bus/pci/devices/{bus}/numa_node").read_text().strip()
    local = Path(f"/sys/bus/pci/devices/{bus}/local_cpulist").read_text().strip()
except OSError as e:
    node = local = f"unreadable ({e})"
import os
print(f"GPU {bus}: numa_node {node}, local cpus {local}; this process may run on {sorted(os.sched_getaffinity(0))}")
for piece in (2 << 20, 32 << 20, H2D):
    PIECE = piece
    t1, t2 = med(h2d), med(d2h)
    print(f"pieces of {piece >> 20} MiB: H2D {H2D / t1 / 1e9:.1f} GB/s, D2H {D2H / t2 / 1e9:.1f} GB/s")
