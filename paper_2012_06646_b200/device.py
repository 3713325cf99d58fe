"""Device-resident operators on torch CUDA tensors (HBM in, HBM out).

The hot path the bench measures: inputs already resident, results left on
the device, everything enqueued on torch's current stream through
``ibc_spread_device`` / ``ibc_interpolate_device``.  torch is plumbing here
(allocation, streams, events); the kernels are libibcuda.so's.
"""
from __future__ import annotations

import ctypes as C

from . import _capi
from ._capi import InvalidArgument, check, load
from .ib import Context, CosineKernel, SpreadWorkspace, StaggeredGrid, _kernel_code


def capture_graph(fn, graph=None):
    """Capture fn() into a CUDA graph with Python's garbage collector paused.

    The library's Python objects (contexts, workspaces, binnings) free device
    memory when collected; a collection that happens to run inside a capture
    would call cudaFree, which is not capturable, and invalidate the whole
    capture.  Collect first, then keep the collector off until the capture
    ends."""
    import gc

    import torch

    graph = graph if graph is not None else torch.cuda.CUDAGraph()
    gc.collect()
    torch.cuda.synchronize()
    enabled = gc.isenabled()
    gc.disable()
    try:
        with torch.cuda.graph(graph):
            fn()
    finally:
        if enabled:
            gc.enable()
    return graph


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(int(t.data_ptr()))


def _require(t, name, numel=None, dtype=None):
    import torch

    dtype = dtype or torch.float64
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidArgument(f"{name} must be a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise InvalidArgument(f"{name} must be contiguous {str(dtype).split('.')[-1]}")
    if numel is not None and t.numel() != numel:
        raise InvalidArgument(f"{name} has {t.numel()} elements, expected {numel}")


def _precision(t):
    """float64 tensors run the FP64 operators, float32 ones the FP32 storage
    mode (ibc_*_device_f32: float in memory, FP64 arithmetic)."""
    import torch

    if isinstance(t, torch.Tensor) and t.dtype == torch.float32:
        return torch.float32, "_f32"
    return torch.float64, ""


class BinnedPoints:
    """ibc_binned: points bucketed for interpolation on one grid."""

    def __init__(self, context: Context):
        h = C.c_void_p()
        check(load().ibc_binned_create(context.handle, C.byref(h)))
        self.handle = h
        self.n = 0
        self.grid = None

    def close(self) -> None:
        if getattr(self, "handle", None):
            load().ibc_binned_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class DeviceOperators:
    """Spread / interpolate on one GPU with a persistent context + workspace."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        self.context = Context(self.device)
        self._ws: dict[tuple, SpreadWorkspace] = {}

    def _sync_stream(self):
        import torch

        self.context.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def workspace(self, n: int, grid: StaggeredGrid) -> SpreadWorkspace:
        key = (n, grid.point_count())
        if key not in self._ws:
            self._ws[key] = SpreadWorkspace(n, grid, 0, context=self.context)
        return self._ws[key]

    def spread(self, points, values, grid: StaggeredGrid, out=None, workspace=None,
               kernel=CosineKernel):
        """points (n, D), values (n,) -> out (prod(extent),), cuda, all float64 --
        or all float32 (the FP32 storage mode, ibc_spread_device_f32)."""
        import torch

        n = points.shape[0] if points.dim() == 2 else points.numel() // grid.dim
        dt, sfx = _precision(points)
        _require(points, "points", n * grid.dim, dt)
        _require(values, "values", n, dt)
        if out is None:
            out = torch.empty(grid.point_count(), dtype=dt, device=points.device)
        _require(out, "out", grid.point_count(), dt)
        ws = workspace if workspace is not None else self.workspace(n, grid)
        self._sync_stream()
        check(getattr(load(), "ibc_spread_device" + sfx)(
            self.context.handle, C.byref(grid.c_grid), _kernel_code(kernel), _ptr(points),
            _ptr(values), n, ws.handle, _ptr(out)))
        ws._mark(n)
        return out

    def interpolate(self, field, points, grid: StaggeredGrid, out=None, kernel=CosineKernel):
        """field (prod(extent),) + points (n, D) -> out (n,), cuda, all float64 --
        or all float32 (the FP32 storage mode, ibc_interpolate_device_f32)."""
        import torch

        n = points.shape[0] if points.dim() == 2 else points.numel() // grid.dim
        dt, sfx = _precision(field)
        _require(field, "field", grid.point_count(), dt)
        _require(points, "points", n * grid.dim, dt)
        if out is None:
            out = torch.empty(n, dtype=dt, device=points.device)
        _require(out, "out", n, dt)
        self._sync_stream()
        check(getattr(load(), "ibc_interpolate_device" + sfx)(
            self.context.handle, C.byref(grid.c_grid), _kernel_code(kernel), _ptr(field),
            _ptr(points), n, _ptr(out)))
        return out

    def bin_points(self, points, grid: StaggeredGrid, kernel=CosineKernel, binned=None):
        """Bin device points for interpolation on `grid` (ibc_bin_points_device):
        the field-independent half of `interpolate`, reusable for any number
        of fields at the same points.  `points` must stay unchanged."""
        n = points.shape[0] if points.dim() == 2 else points.numel() // grid.dim
        dt, sfx = _precision(points)
        _require(points, "points", n * grid.dim, dt)
        b = binned if binned is not None else BinnedPoints(self.context)
        self._sync_stream()
        check(getattr(load(), "ibc_bin_points_device" + sfx)(
            self.context.handle, b.handle, C.byref(grid.c_grid), _kernel_code(kernel),
            _ptr(points), n))
        b.dtype = dt
        b.n, b.grid = n, grid
        b._points = points  # keep the binned tensor alive
        return b

    def interpolate_binned(self, field, binned, out=None):
        """Interpolate `field` at binned points (ibc_interpolate_binned_device)."""
        import torch

        dt = getattr(binned, "dtype", torch.float64)  # the binned points' precision
        sfx = "_f32" if dt == torch.float32 else ""
        _require(field, "field", binned.grid.point_count(), dt)
        if out is None:
            out = torch.empty(binned.n, dtype=dt, device=field.device)
        _require(out, "out", binned.n, dt)
        self._sync_stream()
        check(getattr(load(), "ibc_interpolate_binned_device" + sfx)(
            self.context.handle, binned.handle, _ptr(field), _ptr(out)))
        return out

    @property
    def launches(self) -> int:
        return self.context.launches
