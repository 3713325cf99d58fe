"""Python mirror of the reference operator API, backed by libibcuda.so.

Same names, argument meaning and error behaviour as the reference's header
templates (/root/reference/proj/include/ib/), so tests read like the
reference's own GoogleTest suites:

  reference (C++)                                  here
  ib::StaggeredGrid<D> (grid.hpp:33-83)            StaggeredGrid
  ib::GridField<D> (grid.hpp:85-92)                GridField
  ib::PointSet<D> (grid.hpp:187-188)               (n, D) float64 array
  ib::LagrangianValues (grid.hpp:192)              (n,) float64 array
  ib::CosineKernel (kernel.hpp:31-36)              CosineKernel
  ib::SpreadAlgorithm (spread.hpp:21)              SpreadAlgorithm
  ib::SpreadWorkspace<D> (spread.hpp:27-56)        SpreadWorkspace
  ib::interpolate (interpolate.hpp:22-58)          interpolate
  ib::interpolate_vector (interpolate.hpp:62-72)   interpolate_vector
  ib::spread_serial / _fused / _buffered / _otf    spread_serial / ... (spread.hpp:129-317)
  ib::spread_vector (spread.hpp:321-350)           spread_vector
  ib::stats (stats.hpp)                            stats

std::invalid_argument -> InvalidArgument, std::length_error -> LengthError.
Every operator runs on the B200 through the C ABI; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
import threading

import numpy as np

from . import _capi
from ._capi import InvalidArgument, LengthError, check, load  # noqa: F401

__all__ = [
    "StaggeredGrid", "GridField", "CosineKernel", "Peskin4Kernel", "Roma3Kernel", "Linear2Kernel",
    "KERNELS", "SpreadAlgorithm", "SpreadWorkspace",
    "interpolate", "interpolate_vector", "spread_serial", "spread_fused", "spread_buffered",
    "spread_buffered_otf", "spread_vector", "stats", "Context", "default_context",
    "InvalidArgument", "LengthError",
]


class Context:
    """A device + stream + scratch (ibc_context)."""

    def __init__(self, device: int = 0):
        lib = load()
        h = C.c_void_p()
        check(lib.ibc_context_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)
        self._lib = lib

    def set_stream(self, stream_ptr: int | None) -> None:
        check(self._lib.ibc_context_set_stream(self.handle, C.c_void_p(stream_ptr or 0)))

    def synchronize(self) -> None:
        check(self._lib.ibc_context_synchronize(self.handle))

    def set_spread_path(self, path: str) -> None:
        """'auto' (default), or force 'bank' / 'pull' / 'radix' (ibc_context_set_spread_path)."""
        code = {"auto": _capi.IBC_SPREAD_PATH_AUTO, "bank": _capi.IBC_SPREAD_PATH_BANK,
                "pull": _capi.IBC_SPREAD_PATH_PULL, "radix": _capi.IBC_SPREAD_PATH_RADIX}
        if path not in code:
            raise InvalidArgument(f"unknown spread path {path!r}")
        check(self._lib.ibc_context_set_spread_path(self.handle, code[path]))

    def set_profiling(self, on: bool) -> None:
        check(self._lib.ibc_context_set_profiling(self.handle, int(bool(on))))

    def profile(self) -> dict:
        p = _capi.IbcProfile()
        check(self._lib.ibc_context_get_profile(self.handle, C.byref(p)))
        return {f: getattr(p, f) for f, _ in _capi.IbcProfile._fields_}

    def reset_profile(self) -> None:
        check(self._lib.ibc_context_reset_profile(self.handle))

    @property
    def launches(self) -> int:
        return int(self._lib.ibc_context_launches(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.ibc_context_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


_ctx_lock = threading.Lock()
_contexts: dict[int, Context] = {}


def default_context(device: int | None = None) -> Context:
    if device is None:
        device = int(os.environ.get("IBC_DEVICE", "0"))
    with _ctx_lock:
        if device not in _contexts:
            _contexts[device] = Context(device)
        return _contexts[device]


class StaggeredGrid:
    """ib::StaggeredGrid<D>: x = h*(i + alpha) + origin; validated like the ctor."""

    def __init__(self, extents, spacing, staggering, periodic, origin=None):
        d = len(extents)
        if not (1 <= d <= 3) or len(staggering) != d or len(periodic) != d:
            raise InvalidArgument("grids are 1-, 2-, or 3-dimensional")
        if origin is not None and len(origin) != d:
            raise InvalidArgument("origin must have one entry per axis")
        self._g = _capi.make_grid(extents, spacing, staggering, periodic, origin)
        check(load().ibc_grid_check(C.byref(self._g)))
        self.dim = d
        self.extents = tuple(int(e) for e in extents)
        self._spacing = float(spacing)
        self.staggerings = tuple(float(s) for s in staggering)
        self.periodic = tuple(bool(p) for p in periodic)
        self.origin = tuple(float(o) for o in origin) if origin is not None else (0.0,) * d

    def extent(self, axis: int) -> int:
        return self.extents[axis]

    def spacing(self) -> float:
        return self._spacing

    def staggering(self, axis: int) -> float:
        return self.staggerings[axis]

    def is_periodic(self, axis: int) -> bool:
        return self.periodic[axis]

    def point_count(self) -> int:
        return int(np.prod(self.extents))

    def axis_length(self, axis: int) -> float:
        return self.extents[axis] * self._spacing

    @property
    def c_grid(self) -> _capi.IbcGrid:
        return self._g

    def __eq__(self, other):
        return isinstance(other, StaggeredGrid) and (
            self.extents, self._spacing, self.staggerings, self.periodic, self.origin) == (
            other.extents, other._spacing, other.staggerings, other.periodic, other.origin)

    def __repr__(self):
        return (f"StaggeredGrid(extents={self.extents}, spacing={self._spacing}, "
                f"staggering={self.staggerings}, periodic={self.periodic}, origin={self.origin})")


class GridField:
    """ib::GridField<D>: one value per grid point, colexicographic (axis 0 fastest)."""

    def __init__(self, grid: StaggeredGrid, values=None):
        self.grid = grid
        if values is None:
            self.values = np.zeros(grid.point_count(), np.float64)
        else:
            v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
            if v.size != grid.point_count():
                raise InvalidArgument("field size differs from the grid point count")
            self.values = v


class CosineKernel:
    """ib::CosineKernel: phi(r) = (1 + cos(pi r / 2)) / 4 on |r| < 2, support 4."""

    code = _capi.IBC_KERNEL_COSINE4

    @staticmethod
    def phi(r: float) -> float:
        return 0.0 if not abs(r) < 2.0 else 0.25 * (1.0 + math.cos(0.5 * math.pi * r))

    @staticmethod
    def support() -> int:
        return 4

    @staticmethod
    def radius() -> float:
        return 2.0


class Peskin4Kernel:
    """Peskin's standard 4-point kernel (Peskin 2002, Eq. 6.27), support 4:
    (3 - 2|r| + sqrt(1 + 4|r| - 4r^2)) / 8 on |r| <= 1,
    (5 - 2|r| - sqrt(-7 + 12|r| - 4r^2)) / 8 on 1 < |r| < 2."""

    code = _capi.IBC_KERNEL_PESKIN4

    @staticmethod
    def phi(r: float) -> float:
        a = abs(r)
        if not a < 2.0:
            return 0.0
        if a <= 1.0:
            return (3.0 - 2.0 * a + math.sqrt(1.0 + 4.0 * a - 4.0 * a * a)) * 0.125
        return (5.0 - 2.0 * a - math.sqrt(max(0.0, -7.0 + 12.0 * a - 4.0 * a * a))) * 0.125

    @staticmethod
    def support() -> int:
        return 4

    @staticmethod
    def radius() -> float:
        return 2.0


class Roma3Kernel:
    """The 3-point kernel of Roma, Peskin & Berger (1999), odd support 3
    (cell_index associates the nearest grid point, grid.hpp:121-130):
    (1 + sqrt(1 - 3r^2)) / 3 on |r| <= 1/2,
    (5 - 3|r| - sqrt(1 - 3(1 - |r|)^2)) / 6 on 1/2 < |r| < 3/2."""

    code = _capi.IBC_KERNEL_ROMA3

    @staticmethod
    def phi(r: float) -> float:
        a = abs(r)
        if not a < 1.5:
            return 0.0
        if a <= 0.5:
            return (1.0 + math.sqrt(1.0 - 3.0 * a * a)) / 3.0
        return (5.0 - 3.0 * a - math.sqrt(1.0 - 3.0 * (1.0 - a) * (1.0 - a))) / 6.0

    @staticmethod
    def support() -> int:
        return 3

    @staticmethod
    def radius() -> float:
        return 1.5


class Linear2Kernel:
    """The 2-point hat kernel, 1 - |r| on |r| < 1, support 2."""

    code = _capi.IBC_KERNEL_LINEAR2

    @staticmethod
    def phi(r: float) -> float:
        a = abs(r)
        return 1.0 - a if a < 1.0 else 0.0

    @staticmethod
    def support() -> int:
        return 2

    @staticmethod
    def radius() -> float:
        return 1.0


KERNELS = (CosineKernel, Peskin4Kernel, Roma3Kernel, Linear2Kernel)


class SpreadAlgorithm(enum.IntEnum):
    serial = _capi.IBC_SPREAD_SERIAL
    fused = _capi.IBC_SPREAD_FUSED
    buffered = _capi.IBC_SPREAD_BUFFERED
    otf = _capi.IBC_SPREAD_OTF


def _kernel_code(kernel) -> int:
    """Device kernel id of one of KERNELS (class or instance).  Any other
    Kernel type is rejected: the device evaluates phi itself, so a caller's
    own phi cannot silently be replaced by another kernel's."""
    cls = kernel if isinstance(kernel, type) else type(kernel)
    if cls not in KERNELS:
        raise InvalidArgument(f"unsupported kernel type {cls.__name__}: the device takes "
                              + ", ".join(k.__name__ for k in KERNELS))
    return int(cls.code)


def _points(points, dim: int) -> np.ndarray:
    p = np.ascontiguousarray(points, dtype=np.float64)
    if p.size == 0:
        return p.reshape(0, dim)
    if p.ndim == 1 and dim == 1:
        p = p.reshape(-1, 1)
    if p.ndim != 2 or p.shape[1] != dim:
        raise InvalidArgument(f"points must be an (n, {dim}) array")
    return p


class SpreadWorkspace:
    """ib::SpreadWorkspace<D>(n, grid, b): device buffers sized once.

    After a spread, ``keys`` (sorted), ``perm``, ``run_keys`` and
    ``run_count`` hold the reference's observable results; they are copied
    from the device on first access.
    """

    def __init__(self, n: int, grid: StaggeredGrid, b: int = 0, context: Context | None = None):
        self.context = context or default_context()
        h = C.c_void_p()
        check(load().ibc_workspace_create(self.context.handle, int(n), C.byref(grid.c_grid),
                                          int(b), C.byref(h)))
        self.handle = h
        self.point_count = int(n)
        self.grid_points = grid.point_count()
        self.sweep_width = int(b)
        self._last_n = None

    def _mark(self, n: int) -> None:
        self._last_n = n

    @property
    def run_count(self) -> int:
        q = C.c_size_t()
        check(load().ibc_workspace_run_count(self.handle, C.byref(q)))
        return int(q.value)

    @property
    def keys(self) -> np.ndarray:
        n = self._last_n or 0
        out = np.zeros(n, np.uint32)
        check(load().ibc_workspace_get_keys(self.handle, out.ctypes.data_as(C.c_void_p), n))
        return out

    @property
    def perm(self) -> np.ndarray:
        n = self._last_n or 0
        out = np.zeros(n, np.uint32)
        check(load().ibc_workspace_get_perm(self.handle, out.ctypes.data_as(C.c_void_p), n))
        return out

    @property
    def run_keys(self) -> np.ndarray:
        q = C.c_size_t()
        check(load().ibc_workspace_get_run_keys(self.handle, None, 0, C.byref(q)))
        out = np.zeros(max(q.value, 1), np.uint32)
        check(load().ibc_workspace_get_run_keys(self.handle, out.ctypes.data_as(C.c_void_p),
                                                out.size, C.byref(q)))
        return out[: q.value]

    def close(self) -> None:
        if getattr(self, "handle", None):
            load().ibc_workspace_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _spread(points, values, grid: StaggeredGrid, kernel, algorithm: int, sweep_width: int,
            ws: SpreadWorkspace | None, workers: int, context: Context | None = None) -> GridField:
    p = _points(points, grid.dim)
    v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    ctx = ws.context if ws is not None else (context or default_context())
    out = np.empty(grid.point_count(), np.float64)
    check(load().ibc_spread(ctx.handle, C.byref(grid.c_grid), _kernel_code(kernel), int(algorithm),
                            p.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p),
                            p.shape[0], v.size, int(sweep_width),
                            ws.handle if ws is not None else None, int(workers),
                            out.ctypes.data_as(C.c_void_p)))
    if ws is not None and algorithm in (SpreadAlgorithm.fused, SpreadAlgorithm.buffered):
        ws._mark(p.shape[0])
    return GridField(grid, out)


def spread_serial(points, values, grid: StaggeredGrid, kernel) -> GridField:
    """ib::spread_serial (spread.hpp:129-159): the Algorithm 2 operator."""
    return _spread(points, values, grid, kernel, SpreadAlgorithm.serial, 0, None, 1)


def spread_fused(points, values, grid: StaggeredGrid, kernel, ws: SpreadWorkspace,
                 workers: int = 1) -> GridField:
    """ib::spread_fused (spread.hpp:165-216): key sort + segmented reduce."""
    if ws is None:
        raise InvalidArgument("fused spreading needs a workspace")
    return _spread(points, values, grid, kernel, SpreadAlgorithm.fused, 0, ws, workers)


def spread_buffered(points, values, grid: StaggeredGrid, kernel, ws: SpreadWorkspace,
                    workers: int = 1) -> GridField:
    """ib::spread_buffered (spread.hpp:223-303)."""
    if ws is None:
        raise InvalidArgument("buffered spreading needs a workspace")
    return _spread(points, values, grid, kernel, SpreadAlgorithm.buffered, ws.sweep_width, ws,
                   workers)


def spread_buffered_otf(points, values, grid: StaggeredGrid, kernel, sweep_width: int,
                        workers: int = 1) -> GridField:
    """ib::spread_buffered_otf (spread.hpp:309-317)."""
    return _spread(points, values, grid, kernel, SpreadAlgorithm.otf, sweep_width, None, workers)


def _for_components(count: int, fn) -> list:
    """fn(c) for c < count on one host thread each (ctypes releases the GIL; the
    context serves each host-buffer call on its own lane, so the components'
    copies and kernels overlap).  Raises the lowest component's exception."""
    if count <= 1:
        return [fn(c) for c in range(count)]
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=count - 1) as pool:
        futs = [pool.submit(fn, c) for c in range(count - 1)]
        out, err = [None] * count, [None] * count
        try:
            out[count - 1] = fn(count - 1)
        except Exception as e:  # noqa: BLE001 -- re-raised in component order below
            err[count - 1] = e
        for c, f in enumerate(futs):
            try:
                out[c] = f.result()
            except Exception as e:  # noqa: BLE001
                err[c] = e
    for e in err:
        if e is not None:
            raise e
    return out


def spread_vector(points, values, grids, kernel, algorithm, sweep_width: int,
                  workspace: SpreadWorkspace | None, workers: int = 1):
    """ib::spread_vector (spread.hpp:321-350): one spread per MAC component.

    The reference's per-component argument checks run first, in its order; the
    components before the first failing one then run concurrently
    (_for_components) and its error is raised.  With a workspace the last
    component spreads through it (so it holds that component's sort, as in the
    reference); the others run the same device operator on its context."""
    grids = list(grids)
    dim = grids[0].dim if grids else 0
    if len(grids) != dim:
        raise InvalidArgument("expected one grid per vector component")
    n = _points(points, dim).shape[0] if dim else 0
    ok, fail = dim, None
    for c in range(dim):
        try:
            nv = np.asarray(values[c]).size
            if algorithm in (SpreadAlgorithm.fused, SpreadAlgorithm.buffered):
                if workspace is None:
                    raise InvalidArgument("fused spreading needs a workspace"
                                          if algorithm == SpreadAlgorithm.fused
                                          else "buffered spreading needs a workspace")
            elif algorithm == SpreadAlgorithm.otf:
                if sweep_width < 1:
                    raise InvalidArgument("sweep width must be >= 1")
            elif algorithm != SpreadAlgorithm.serial:
                raise InvalidArgument("unknown spreading algorithm")
            if nv != n:
                raise InvalidArgument("one value per point required")
            if not 1 <= kernel.support() <= 8:
                raise InvalidArgument("unsupported kernel support size")
            if workspace is not None and algorithm in (SpreadAlgorithm.fused, SpreadAlgorithm.buffered):
                if workspace.point_count != n:
                    raise InvalidArgument("workspace sized for a different point count")
                if workspace.grid_points != grids[c].point_count():
                    raise InvalidArgument("workspace sized for a different grid")
                if algorithm == SpreadAlgorithm.buffered and workspace.sweep_width < 1:
                    raise InvalidArgument("workspace has no sweep buffers")
        except InvalidArgument as e:
            ok, fail = c, e
            break
    ctx = workspace.context if workspace is not None else None

    def component(c):
        last = c == dim - 1
        if algorithm == SpreadAlgorithm.serial or (not last and algorithm != SpreadAlgorithm.otf):
            return _spread(points, values[c], grids[c], kernel, SpreadAlgorithm.serial, 0, None, 1,
                           context=ctx)
        if algorithm == SpreadAlgorithm.fused:
            return spread_fused(points, values[c], grids[c], kernel, workspace, workers)
        if algorithm == SpreadAlgorithm.buffered:
            return spread_buffered(points, values[c], grids[c], kernel, workspace, workers)
        return spread_buffered_otf(points, values[c], grids[c], kernel, sweep_width, workers)

    out = _for_components(ok, component)
    if fail is not None:
        raise fail
    return out


def interpolate(field: GridField, points, kernel, workers: int = 1) -> np.ndarray:
    """ib::interpolate (interpolate.hpp:22-58): E_i = h^d sum delta_h(x_k - X_i) e_k."""
    grid = field.grid
    p = _points(points, grid.dim)
    f = np.ascontiguousarray(field.values, dtype=np.float64)
    out = np.empty(p.shape[0], np.float64)
    ctx = default_context()
    check(load().ibc_interpolate(ctx.handle, C.byref(grid.c_grid), _kernel_code(kernel),
                                 f.ctypes.data_as(C.c_void_p), p.ctypes.data_as(C.c_void_p),
                                 p.shape[0], int(workers), out.ctypes.data_as(C.c_void_p)))
    return out


def interpolate_vector(fields, points, kernel, workers: int = 1):
    """ib::interpolate_vector (interpolate.hpp:62-72)."""
    fields = list(fields)
    dim = fields[0].grid.dim if fields else 0
    if len(fields) != dim:
        raise InvalidArgument("expected one field per vector component")
    # the components concurrently (_for_components); each call checks its
    # arguments before any work, like the reference's
    return _for_components(dim, lambda c: interpolate(fields[c], points, kernel, workers))


class stats:
    """ib::stats (stats.hpp:9-25): n_points * s^d per operation."""

    @staticmethod
    def delta_evaluations() -> int:
        return int(load().ibc_delta_evaluations())

    @staticmethod
    def reset_delta_evaluations() -> None:
        load().ibc_reset_delta_evaluations()
