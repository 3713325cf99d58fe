"""Parity oracle for the IB spread/interpolate path -- TEST INFRASTRUCTURE ONLY.

Two CPU implementations sit behind this module:

* ``liboracle.so`` -- ``ib_oracle.c``, a plain-C restatement of the reference
  algorithms (every function cites /root/reference/proj/include/ib/file:line).
* ``_ref/libibref.so`` -- the reference headers themselves, compiled in place
  by ``oracle/Makefile`` (present when /root/reference was available at build
  time; the prebuilt .so travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package.  The product library never does.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


class OrGrid(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("extent", C.c_int * 3),
        ("spacing", C.c_double),
        ("staggering", C.c_double * 3),
        ("periodic", C.c_int * 3),
        ("origin", C.c_double * 3),
    ]


def make_grid(extents, spacing, staggering, periodic, origin=None) -> OrGrid:
    d = len(extents)
    g = OrGrid()
    g.dim = d
    for a in range(3):
        g.extent[a] = int(extents[a]) if a < d else 1
        g.staggering[a] = float(staggering[a]) if a < d else 0.0
        g.periodic[a] = int(bool(periodic[a])) if a < d else 0
        g.origin[a] = float(origin[a]) if (origin is not None and a < d) else 0.0
    g.spacing = float(spacing)
    return g


def grid_points(g: OrGrid) -> int:
    p = 1
    for a in range(g.dim):
        p *= g.extent[a]
    return p


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_G = C.POINTER(OrGrid)
_sz = C.c_size_t


def _load(path: Path, sigs: dict):
    lib = C.CDLL(str(path))
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_ORACLE_SIGS = {
    "or_grid_check": (C.c_int, [_G]),
    "or_cell_key": (C.c_uint32, [_G, C.POINTER(C.c_int)]),
    "or_cell_index": (None, [_G, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int)]),
    "or_wrap_position": (None, [_G, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "or_grid_index": (C.c_uint32, [_G, C.POINTER(C.c_int)]),
    "or_cell_key_inverse": (None, [_G, C.c_uint32, C.POINTER(C.c_int)]),
    "or_cosine_phi": (C.c_double, [C.c_double]),
    "or_shift": (None, [C.c_int, C.c_int64, C.c_int, C.POINTER(C.c_int)]),
    "or_key_value_sort": (None, [_up, _up, _sz]),
    "or_segmented_reduce": (_sz, [_up, _dp, _sz, _up, _dp]),
    "or_prepare_keys": (_sz, [_G, _dp, _sz, _up, _up, _up]),
    "or_kernel_support": (C.c_int, [C.c_int]),
    "or_kernel_phi": (C.c_double, [C.c_int, C.c_double]),
    "or_prepare_keys_k": (_sz, [_G, C.c_int, _dp, _sz, _up, _up, _up]),
    "or_spread_serial_k": (C.c_int, [_G, C.c_int, _dp, _dp, _sz, _dp]),
    "or_spread_fused_k": (C.c_int, [_G, C.c_int, _dp, _dp, _sz, _dp, _up, _up, _up, C.POINTER(_sz)]),
    "or_interpolate_k": (C.c_int, [_G, C.c_int, _dp, _dp, _sz, _dp]),
    "or_spread_serial": (C.c_int, [_G, _dp, _dp, _sz, _dp]),
    "or_spread_fused": (C.c_int, [_G, _dp, _dp, _sz, _dp, _up, _up, _up, C.POINTER(_sz)]),
    "or_interpolate": (C.c_int, [_G, _dp, _dp, _sz, _dp]),
    "or_scatter_points": (None, [C.c_uint64, C.c_double, C.c_uint64, _dp]),
    "or_home_cells": (None, [_G, _dp, _sz, C.c_int, C.c_int,
                             np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")]),
}

_REF_SIGS = {
    "ref_spread": (C.c_int, [C.c_int, _G, _dp, _dp, _sz, C.c_int, C.c_int, _dp,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_sz)]),
    "ref_interpolate": (C.c_int, [_G, _dp, _dp, _sz, C.c_int, _dp]),
    "ref_spread_k": (C.c_int, [C.c_int, C.c_int, _G, _dp, _dp, _sz, C.c_int, C.c_int, _dp,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_sz)]),
    "ref_interpolate_k": (C.c_int, [C.c_int, _G, _dp, _dp, _sz, C.c_int, _dp]),
    "ref_cell_keys": (C.c_int, [_G, _dp, _sz, _up]),
    "ref_grid_check": (C.c_int, [_G]),
    "ref_key_value_sort": (None, [_up, _up, _sz, C.c_int]),
    "ref_segmented_reduce": (_sz, [_up, _dp, _sz, C.c_int, _up, _dp]),
    "ref_scatter_points": (None, [C.c_uint64, C.c_double, C.c_uint64, _dp]),
    "ref_delta_evaluations": (C.c_uint64, []),
    "ref_reset_delta_evaluations": (None, []),
    "ref_time_step": (C.c_int, [_G, _dp, _dp, _dp, _dp, _sz, C.c_int, C.c_int, _dp, _dp]),
    "ref_run_verification": (C.c_int, [C.c_uint64, C.c_int, C.c_int]),
}

_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        p = HERE / "liboracle.so"
        if not p.exists():
            raise RuntimeError(f"oracle not built: {p} (run `make -C oracle`)")
        _lib = _load(p, _ORACLE_SIGS)
    return _lib


def ref_available() -> bool:
    return (HERE / "_ref" / "libibref.so").exists()


def ref():
    global _ref
    if _ref is None:
        p = HERE / "_ref" / "libibref.so"
        if not p.exists():
            raise RuntimeError(f"reference build absent: {p}")
        _ref = _load(p, _REF_SIGS)
    return _ref


def _pts(points, d):
    p = np.ascontiguousarray(points, dtype=np.float64).reshape(-1)
    assert p.size % d == 0
    return p


# ---------------------------------------------------------------- C restatement
# Kernel ids (include/ibcuda.h ibc_kernel): 0 cosine (the reference's
# CosineKernel), 1 Peskin 4-point, 2 Roma 3-point, 3 hat.
KERNELS = {"cosine4": 0, "peskin4": 1, "roma3": 2, "linear2": 3}


def kernel_phi(kernel, r):
    return lib().or_kernel_phi(int(kernel), float(r))


def prepare_keys(g, points, kernel=0):
    p = _pts(points, g.dim)
    n = p.size // g.dim
    keys = np.zeros(max(n, 1), np.uint32)
    perm = np.zeros(max(n, 1), np.uint32)
    run = np.zeros(max(n, 1), np.uint32)
    q = lib().or_prepare_keys_k(C.byref(g), int(kernel), p, n, keys, perm, run)
    return keys[:n], perm[:n], run[:q]


def spread_serial(g, points, values, kernel=0):
    p = _pts(points, g.dim)
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = np.zeros(grid_points(g), np.float64)
    lib().or_spread_serial_k(C.byref(g), int(kernel), p, v, v.size, out)
    return out


def spread_fused(g, points, values, kernel=0):
    """Returns (field, keys, perm, run_keys) exactly as ws.* after spread_fused."""
    p = _pts(points, g.dim)
    v = np.ascontiguousarray(values, dtype=np.float64)
    n = v.size
    out = np.zeros(grid_points(g), np.float64)
    keys = np.zeros(max(n, 1), np.uint32)
    perm = np.zeros(max(n, 1), np.uint32)
    run = np.zeros(max(n, 1), np.uint32)
    q = _sz(0)
    lib().or_spread_fused_k(C.byref(g), int(kernel), p, v, n, out, keys, perm, run, C.byref(q))
    return out, keys[:n], perm[:n], run[: q.value]


def interpolate(g, field, points, kernel=0):
    p = _pts(points, g.dim)
    f = np.ascontiguousarray(field, dtype=np.float64)
    n = p.size // g.dim
    out = np.zeros(n, np.float64)
    lib().or_interpolate_k(C.byref(g), int(kernel), f, p, n, out)
    return out


def home_cells(g, points, wrap=True, support=4):
    """cell_index(wrap_position(x)) with periodic axes wrapped into [0, n)
    (grid.hpp:121-151, 197-207): the home cell of every point, (n, dim) ints.
    wrap=False leaves the cell unwrapped (it can equal n on a periodic axis)."""
    p = _pts(points, g.dim)
    n = p.size // g.dim
    out = np.zeros(max(n, 1) * g.dim, np.int32)
    lib().or_home_cells(C.byref(g), p, n, int(support), 1 if wrap else 0, out)
    return out[: n * g.dim].reshape(n, g.dim).astype(np.int64)


def scatter_points(n, edge, seed):
    out = np.zeros(n * 3, np.float64)
    lib().or_scatter_points(n, edge, seed, out)
    return out.reshape(n, 3)


# ---------------------------------------------------------------- reference build
def ref_spread(g, points, values, algo="fused", workers=1, sweep_width=8, kernel=0):
    codes = {"serial": 0, "fused": 1, "buffered": 2, "otf": 3}
    p = _pts(points, g.dim)
    v = np.ascontiguousarray(values, dtype=np.float64)
    n = v.size
    out = np.zeros(grid_points(g), np.float64)
    keys = np.zeros(max(n, 1), np.uint32)
    perm = np.zeros(max(n, 1), np.uint32)
    run = np.zeros(max(n, 1), np.uint32)
    q = _sz(0)
    rc = ref().ref_spread_k(int(kernel), codes[algo], C.byref(g), p, v, n, workers, sweep_width,
                            out, keys.ctypes.data, perm.ctypes.data, run.ctypes.data, C.byref(q))
    if rc:
        raise ValueError(f"reference spread failed with code {rc}")
    return out, keys[:n], perm[:n], run[: q.value]


def ref_interpolate(g, field, points, workers=1, kernel=0):
    p = _pts(points, g.dim)
    f = np.ascontiguousarray(field, dtype=np.float64)
    n = p.size // g.dim
    out = np.zeros(n, np.float64)
    rc = ref().ref_interpolate_k(int(kernel), C.byref(g), f, p, n, workers, out)
    if rc:
        raise ValueError(f"reference interpolate failed with code {rc}")
    return out


def ref_time_step(g, x_star, values, x_n, field, workers, reps):
    n = np.asarray(values).size
    ts = np.zeros(reps)
    ti = np.zeros(reps)
    rc = ref().ref_time_step(C.byref(g), _pts(x_star, g.dim), np.ascontiguousarray(values, np.float64),
                             _pts(x_n, g.dim), np.ascontiguousarray(field, np.float64), n,
                             workers, reps, ts, ti)
    if rc:
        raise ValueError(f"reference step failed with code {rc}")
    return ts, ti


def max_rel_deviation(got, want):
    """inc/bench/verify.hpp:36-45: max|got-want| / max|want| (1 if want == 0)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    scale = float(np.max(np.abs(want))) if want.size else 0.0
    if scale == 0.0:
        scale = 1.0
    dev = float(np.max(np.abs(got - want))) if got.size else 0.0
    return dev / scale


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1
