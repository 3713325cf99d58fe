"""Diagnostic: concurrent pinned host-buffer calls through the C ABI (one-off)."""
import ctypes as C
import threading
import time

import numpy as np
import torch

from paper_2012_06646_b200 import _capi, ib, synth

N, n = 256, 1 << 20
data = synth.config2()
g = ib.StaggeredGrid([N] * 3, data["h"], [0.5, 0.5, 0.0], [True] * 3)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hx_s, hx_n, hg, hf = pin(data["x_star"]), pin(data["x_n"]), pin(data["values"]), pin(data["field"])
h_ell = torch.empty(N ** 3, dtype=torch.float64).pin_memory()
h_E = torch.empty(n, dtype=torch.float64).pin_memory()
lib = _capi.load()
ctx = ib.default_context(0)
ws = ib.SpreadWorkspace(n, g, context=ctx)
vp = lambda t: C.c_void_p(t.data_ptr())
log = []


def sp():
    t0 = time.perf_counter()
    _capi.check(lib.ibc_spread(ctx.handle, C.byref(g.c_grid), 0, 1, vp(hx_s), vp(hg), n, n, 0,
                               ws.handle, 0, vp(h_ell)))
    log.append(("spread", t0, time.perf_counter()))


def it():
    t0 = time.perf_counter()
    _capi.check(lib.ibc_interpolate(ctx.handle, C.byref(g.c_grid), 0, vp(hf), vp(hx_n), n, 0, vp(h_E)))
    log.append(("interp", t0, time.perf_counter()))


for mode in ("seq", "conc", "seq", "conc", "conc", "spread-only", "interp-only"):
    log.clear()
    T0 = time.perf_counter()
    if mode == "seq":
        sp(); it()
    elif mode == "conc":
        th = threading.Thread(target=it); th.start(); sp(); th.join()
    elif mode == "spread-only":
        sp()
    else:
        it()
    T1 = time.perf_counter()
    print(f"{mode:12s} {1e3*(T1-T0):7.2f} ms", [(k, round(1e3*(a-T0), 2), round(1e3*(b-T0), 2)) for k, a, b in log])
