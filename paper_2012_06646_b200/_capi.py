"""ctypes binding of the C ABI in include/ibcuda.h (libibcuda.so).

This is the binding a Python caller of the reference-facing boundary would
add; INTEGRATION.md shows it next to the C++ (include/ib_b200/ib.hpp) one.
The library is required: there is no CPU fallback, and importing the
operators without the built extension raises immediately.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libibcuda.so"

IBC_OK = 0
IBC_ERR_INVALID_ARGUMENT = 1
IBC_ERR_LENGTH = 2
IBC_ERR_CUDA = 3
IBC_ERR_ALLOC = 4

IBC_KERNEL_COSINE4 = 0
IBC_KERNEL_PESKIN4 = 1
IBC_KERNEL_ROMA3 = 2
IBC_KERNEL_LINEAR2 = 3

IBC_SPREAD_SERIAL = 0
IBC_SPREAD_FUSED = 1
IBC_SPREAD_BUFFERED = 2
IBC_SPREAD_OTF = 3

IBC_SPREAD_PATH_AUTO = 0
IBC_SPREAD_PATH_BANK = 1
IBC_SPREAD_PATH_PULL = 2
IBC_SPREAD_PATH_RADIX = 3


class IbcGrid(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("extent", C.c_int * 3),
        ("spacing", C.c_double),
        ("staggering", C.c_double * 3),
        ("periodic", C.c_int * 3),
        ("origin", C.c_double * 3),
    ]


class IbcProfile(C.Structure):
    _fields_ = [
        ("keys_ms", C.c_double),
        ("sort_ms", C.c_double),
        ("rows_ms", C.c_double),
        ("prep_ms", C.c_double),
        ("spread_ms", C.c_double),
        ("interp_ms", C.c_double),
        ("spread_calls", C.c_uint64),
        ("interp_calls", C.c_uint64),
    ]


class IbcSlab(C.Structure):
    _fields_ = [
        ("z_first", C.c_int),
        ("nz_global", C.c_int),
        ("periodic_global", C.c_int),
    ]


class IbcSlabLink(C.Structure):
    _fields_ = [
        ("nloc", C.c_int),
        ("nloc_down", C.c_int),
        ("plane", C.c_size_t),
        ("has_down", C.c_int),
        ("has_up", C.c_int),
        ("d_local", C.c_void_p),
        ("d_down", C.c_void_p),
        ("d_up", C.c_void_p),
        ("d_sig", C.c_void_p),
        ("d_sig_down", C.c_void_p),
        ("d_sig_up", C.c_void_p),
    ]


class IbcIpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64)]


_vp = C.c_void_p
_sz = C.c_size_t
_G = C.POINTER(IbcGrid)
_st = C.c_int

# name -> (restype, argtypes); every symbol declared in include/ibcuda.h.
SIGNATURES = {
    "ibc_version": (C.c_int, []),
    "ibc_last_error": (C.c_char_p, []),
    "ibc_context_create": (_st, [C.c_int, C.POINTER(_vp)]),
    "ibc_context_destroy": (_st, [_vp]),
    "ibc_context_set_stream": (_st, [_vp, _vp]),
    "ibc_context_synchronize": (_st, [_vp]),
    "ibc_context_set_profiling": (_st, [_vp, C.c_int]),
    "ibc_context_get_profile": (_st, [_vp, C.POINTER(IbcProfile)]),
    "ibc_context_reset_profile": (_st, [_vp]),
    "ibc_context_launches": (C.c_uint64, [_vp]),
    "ibc_context_set_spread_path": (_st, [_vp, C.c_int]),
    "ibc_grid_check": (_st, [_G]),
    "ibc_workspace_create": (_st, [_vp, _sz, _G, C.c_int, C.POINTER(_vp)]),
    "ibc_workspace_destroy": (_st, [_vp]),
    "ibc_workspace_info": (_st, [_vp, C.POINTER(_sz), C.POINTER(_sz), C.POINTER(C.c_int)]),
    "ibc_workspace_run_count": (_st, [_vp, C.POINTER(_sz)]),
    "ibc_workspace_get_keys": (_st, [_vp, _vp, _sz]),
    "ibc_workspace_get_perm": (_st, [_vp, _vp, _sz]),
    "ibc_workspace_get_run_keys": (_st, [_vp, _vp, _sz, C.POINTER(_sz)]),
    "ibc_spread": (_st, [_vp, _G, C.c_int, C.c_int, _vp, _vp, _sz, _sz, C.c_int, _vp, C.c_int, _vp]),
    "ibc_interpolate": (_st, [_vp, _G, C.c_int, _vp, _vp, _sz, C.c_int, _vp]),
    "ibc_spread_device": (_st, [_vp, _G, C.c_int, _vp, _vp, _sz, _vp, _vp]),
    "ibc_interpolate_device": (_st, [_vp, _G, C.c_int, _vp, _vp, _sz, _vp]),
    "ibc_spread_f32": (_st, [_vp, _G, C.c_int, C.c_int, _vp, _vp, _sz, _sz, C.c_int, _vp, C.c_int, _vp]),
    "ibc_interpolate_f32": (_st, [_vp, _G, C.c_int, _vp, _vp, _sz, C.c_int, _vp]),
    "ibc_spread_device_f32": (_st, [_vp, _G, C.c_int, _vp, _vp, _sz, _vp, _vp]),
    "ibc_interpolate_device_f32": (_st, [_vp, _G, C.c_int, _vp, _vp, _sz, _vp]),
    "ibc_bin_points_device_f32": (_st, [_vp, _vp, _G, C.c_int, _vp, _sz]),
    "ibc_interpolate_binned_device_f32": (_st, [_vp, _vp, _vp, _vp]),
    "ibc_spread_slab_device": (_st, [_vp, _G, C.POINTER(IbcSlab), C.c_int, _vp, _vp, _sz, _vp, _vp]),
    "ibc_interpolate_slab_device": (_st, [_vp, _G, C.POINTER(IbcSlab), C.c_int, _vp, _vp, _sz, _vp]),
    "ibc_home_planes_device": (_st, [_vp, _G, C.c_int, _vp, _sz, _vp]),
    "ibc_kernel_support": (C.c_int, [C.c_int]),
    "ibc_key_value_sort": (_st, [_vp, _vp, _vp, _sz, _sz, C.c_int]),
    "ibc_key_value_sort_device": (_st, [_vp, _vp, _vp, _sz, _sz]),
    "ibc_segmented_reduce_rows": (_st, [_vp, _vp, _vp, _sz, _sz, _vp, _sz, _vp, _sz, C.c_int,
                                        C.POINTER(_sz)]),
    "ibc_count_unique": (_st, [_vp, _vp, _sz, C.c_int, C.POINTER(_sz)]),
    "ibc_collect_unique_keys": (_st, [_vp, _vp, _sz, _vp, _sz, C.POINTER(_sz)]),
    "ibc_add_delta_evaluations": (None, [C.c_uint64]),
    "ibc_fnv1a": (C.c_uint64, [_vp, _sz, C.c_uint64]),
    "ibc_device_alloc": (_st, [_vp, _sz, C.POINTER(_vp)]),
    "ibc_device_free": (_st, [_vp, _vp]),
    "ibc_ipc_get_handle": (_st, [_vp, _vp, C.POINTER(IbcIpcHandle)]),
    "ibc_ipc_open_handle": (_st, [_vp, C.POINTER(IbcIpcHandle), C.POINTER(_vp)]),
    "ibc_ipc_close_handle": (_st, [_vp, _vp]),
    "ibc_slab_signals_create": (_st, [_vp, C.POINTER(_vp)]),
    "ibc_slab_ghost_sum_device": (_st, [_vp, C.POINTER(IbcSlabLink), C.c_uint64]),
    "ibc_slab_halo_fill_device": (_st, [_vp, C.POINTER(IbcSlabLink), C.c_uint64]),
    "ibc_slab_link_error": (_st, [_vp, C.POINTER(IbcSlabLink), C.POINTER(C.c_int)]),
    "ibc_binned_create": (_st, [_vp, C.POINTER(_vp)]),
    "ibc_binned_destroy": (_st, [_vp]),
    "ibc_bin_points_device": (_st, [_vp, _vp, _G, C.c_int, _vp, _sz]),
    "ibc_interpolate_binned_device": (_st, [_vp, _vp, _vp, _vp]),
    "ibc_delta_evaluations": (C.c_uint64, []),
    "ibc_reset_delta_evaluations": (None, []),
}


class IbError(RuntimeError):
    """Base of the errors raised through the C ABI."""


class InvalidArgument(IbError, ValueError):
    """std::invalid_argument in the reference."""


class LengthError(IbError, ValueError):
    """std::length_error in the reference."""


class CudaError(IbError):
    """A CUDA runtime failure inside the library."""


class AllocationError(IbError, MemoryError):
    """std::bad_alloc (workspace construction)."""


_ERRORS = {
    IBC_ERR_INVALID_ARGUMENT: InvalidArgument,
    IBC_ERR_LENGTH: LengthError,
    IBC_ERR_CUDA: CudaError,
    IBC_ERR_ALLOC: AllocationError,
}

_lib = None


def load(path: Path | None = None):
    """Load libibcuda.so (in-tree build).  Raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 IB operators)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(status: int) -> None:
    if status == IBC_OK:
        return
    msg = (_lib or load()).ibc_last_error().decode(errors="replace")
    raise _ERRORS.get(status, IbError)(msg)


def make_grid(extents, spacing, staggering, periodic, origin=None) -> IbcGrid:
    d = len(extents)
    g = IbcGrid()
    g.dim = d
    for a in range(3):
        g.extent[a] = int(extents[a]) if a < d else 1
        g.staggering[a] = float(staggering[a]) if a < d else 0.0
        g.periodic[a] = int(bool(periodic[a])) if a < d else 0
        g.origin[a] = float(origin[a]) if (origin is not None and a < d) else 0.0
    g.spacing = float(spacing)
    return g
