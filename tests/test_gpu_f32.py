"""FP32 storage mode (ibc_*_f32; SURVEY 8(b) precision F32) on the B200.

Float inputs are widened exactly to double on the device and run through the
FP64 operators, so the float result must be the FP64 operator's result on the
widened inputs rounded once -- bit for bit -- and within the north_star's
float tolerance (1e-5; here 1e-6) of the oracle on those inputs.
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_2012_06646_b200 import _capi, ib
from paper_2012_06646_b200.device import DeviceOperators

pytestmark = pytest.mark.gpu
TOL32 = 1e-6  # float results vs the FP64 oracle (north_star: 1e-5 in float)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def og(g):
    return O.make_grid(g.extents, g.spacing(), g.staggerings, g.periodic, g.origin)


def rand32(g, n, rng):
    pts = np.empty((n, g.dim))
    for a in range(g.dim):
        L = g.axis_length(a)
        pts[:, a] = g.origin[a] + (rng.uniform(-0.5 * L, 1.5 * L, n) if g.is_periodic(a)
                                   else rng.uniform(0, L, n))
    return pts.astype(np.float32)


CASES = [  # (extents, periodic, kernel id): TMA gather + bank sweep, closed axes, generic paths
    ([64, 64, 64], [True] * 3, 0),
    ([256, 64, 48], [True] * 3, 0),   # box-mode TMA planes for float (nx % 256 == 0)
    ([64, 48, 40], [False, True, False], 0),
    ([40, 36, 24], [True] * 3, 1),    # Peskin 4-point; nx % 16 != 0: generic gather
    ([32, 32, 32], [True] * 3, 2),    # Roma 3-point (odd support): radix + tiles
    ([48, 40], [True, False], 0),     # 2-D
]
KERNEL_OF = [ib.CosineKernel(), ib.Peskin4Kernel(), ib.Roma3Kernel(), ib.Linear2Kernel()]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_f32_device_is_the_fp64_operator_rounded_once(torch_cuda, case):
    torch = torch_cuda
    ext, per, k = CASES[case]
    kern = KERNEL_OF[k]
    rng = np.random.default_rng(40 + case)
    g = ib.StaggeredGrid(ext, 0.5, [0.5, 0.5, 0.0][: len(ext)], per)
    n = 30000
    pts = rand32(g, n, rng)
    vals = rng.uniform(-1, 1, n).astype(np.float32)
    field = rng.uniform(-1, 1, g.point_count()).astype(np.float32)
    ops = DeviceOperators(0)
    dev = lambda a: torch.from_numpy(a).cuda()
    p32, v32, f32 = dev(pts), dev(vals), dev(field)
    s32 = ops.spread(p32, v32, g, kernel=kern)
    e32 = ops.interpolate(f32, p32, g, kernel=kern)
    s64 = ops.spread(p32.double(), v32.double(), g, kernel=kern)
    e64 = ops.interpolate(f32.double(), p32.double(), g, kernel=kern)
    torch.cuda.synchronize()
    assert s32.dtype == torch.float32 and e32.dtype == torch.float32
    assert torch.equal(s32, s64.float()) and torch.equal(e32, e64.float())
    og_ = og(g)
    want_s = O.spread_serial(og_, pts.astype(np.float64), vals.astype(np.float64), kernel=k)
    want_e = O.interpolate(og_, field.astype(np.float64), pts.astype(np.float64), kernel=k)
    assert O.max_rel_deviation(s32.cpu().numpy().astype(np.float64), want_s) <= TOL32
    assert O.max_rel_deviation(e32.cpu().numpy().astype(np.float64), want_e) <= TOL32


def test_f32_config2_full_size(torch_cuda):
    torch = torch_cuda
    from paper_2012_06646_b200 import synth

    N, n, edge = 256, 1 << 20, 16e-4
    h = edge / N
    g = ib.StaggeredGrid([N] * 3, h, [0.5, 0.5, 0.0], [True] * 3)
    pts = synth.scatter_points(n, edge, 1).astype(np.float32)
    vals = synth.uniform_pm1(n, 2).astype(np.float32)
    field = synth.uniform_pm1(N ** 3, 4).astype(np.float32)
    ops = DeviceOperators(0)
    p32 = torch.from_numpy(pts).cuda()
    v32, f32 = torch.from_numpy(vals).cuda(), torch.from_numpy(field).cuda()
    s32, e32 = ops.spread(p32, v32, g), ops.interpolate(f32, p32, g)
    s64, e64 = ops.spread(p32.double(), v32.double(), g), ops.interpolate(f32.double(), p32.double(), g)
    assert torch.equal(s32, s64.float()) and torch.equal(e32, e64.float())
    sub = slice(0, 20000)
    og_ = og(g)
    want_e = O.interpolate(og_, field.astype(np.float64), pts[sub].astype(np.float64))
    assert O.max_rel_deviation(e32[sub].cpu().numpy().astype(np.float64), want_e) <= TOL32


def test_f32_host_buffers_and_workspace(torch_cuda):
    # ibc_spread_f32 / ibc_interpolate_f32 (host buffers, pageable): keys and
    # permutation of the workspace bit-exact, values within the float bar
    rng = np.random.default_rng(7)
    g = ib.StaggeredGrid([64, 64, 32], 0.25, [0.5, 0.5, 0.0], [True] * 3)
    n = 20000
    pts = rand32(g, n, rng)
    vals = rng.uniform(-1, 1, n).astype(np.float32)
    field = rng.uniform(-1, 1, g.point_count()).astype(np.float32)
    lib = _capi.load()
    ctx = ib.default_context()
    ws = ib.SpreadWorkspace(n, g)
    out = np.empty(g.point_count(), np.float32)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    _capi.check(lib.ibc_spread_f32(ctx.handle, C.byref(g.c_grid), _capi.IBC_KERNEL_COSINE4,
                                   _capi.IBC_SPREAD_FUSED, vp(pts), vp(vals), n, n, 0, ws.handle,
                                   1, vp(out)))
    ws._mark(n)  # (the raw C call bypasses ib.spread_fused's bookkeeping)
    E = np.empty(n, np.float32)
    _capi.check(lib.ibc_interpolate_f32(ctx.handle, C.byref(g.c_grid), _capi.IBC_KERNEL_COSINE4,
                                        vp(field), vp(pts), n, 1, vp(E)))
    og_ = og(g)
    want, keys, perm, runs = O.spread_fused(og_, pts.astype(np.float64), vals.astype(np.float64))
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert ws.run_count == len(runs)
    assert O.max_rel_deviation(out.astype(np.float64), want) <= TOL32
    want_e = O.interpolate(og_, field.astype(np.float64), pts.astype(np.float64))
    assert O.max_rel_deviation(E.astype(np.float64), want_e) <= TOL32
    # the FP64 host entry point on the widened inputs, rounded once
    ref = ib.spread_fused(pts.astype(np.float64), vals.astype(np.float64), g, ib.CosineKernel(), ws, 1)
    assert np.array_equal(out, ref.values.astype(np.float32))


def test_f32_rejects_mixed_precision(torch_cuda):
    torch = torch_cuda
    g = ib.StaggeredGrid([32, 32, 32], 0.5, [0.5, 0.5, 0.0], [True] * 3)
    ops = DeviceOperators(0)
    p = torch.zeros((10, 3), dtype=torch.float32, device="cuda")
    with pytest.raises(ib.InvalidArgument):
        ops.spread(p, torch.zeros(10, dtype=torch.float64, device="cuda"), g)
    with pytest.raises(ib.InvalidArgument):
        ops.interpolate(torch.zeros(g.point_count(), dtype=torch.float32, device="cuda"),
                        p.double(), g)


def test_f32_binned_equals_unbinned(torch_cuda):
    # ibc_bin_points_device_f32 / ibc_interpolate_binned_device_f32: the same
    # results as ibc_interpolate_device_f32, bit for bit, for several fields
    torch = torch_cuda
    rng = np.random.default_rng(9)
    for ext, per in (([64, 48, 40], [True] * 3), ([40, 36, 24], [False, True, True])):
        g = ib.StaggeredGrid(ext, 0.25, [0.5, 0.5, 0.0], per)
        pts = torch.from_numpy(rand32(g, 20000, rng)).cuda()
        ops = DeviceOperators(0)
        b = ops.bin_points(pts, g)
        for s in range(3):
            f = torch.from_numpy(rng.uniform(-1, 1, g.point_count()).astype(np.float32)).cuda()
            assert torch.equal(ops.interpolate_binned(f, b), ops.interpolate(f, pts, g))
