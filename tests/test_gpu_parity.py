"""CUDA path vs the pinned oracle and the reference's golden vectors (B200).

Mirrors the reference's own suites (tests/coupling_test.cpp, grid_test.cpp,
primitives_test.cpp, inc/bench/verify.hpp).  Bar: sort keys, permutations and
run keys bit-exact; values within the reference's max_rel_deviation <= 1e-12
(inc/bench/verify.hpp:36-45; reduction order and cos rounding differ).
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2012_06646_b200 import ib

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
K = ib.CosineKernel()
TOL = 1e-12  # FP64 tolerance (north_star; verify.hpp:148)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rand_points(g, n, rng):
    pts = np.empty((n, g.dim))
    for a in range(g.dim):
        L = g.axis_length(a)
        pts[:, a] = g.origin[a] + (rng.uniform(-L, 2 * L, n) if g.is_periodic(a) else rng.uniform(0, L, n))
    return pts


def og(g):
    return O.make_grid(g.extents, g.spacing(), g.staggerings, g.periodic, g.origin)


# ------------------------------------------------------------------ golden vectors
def test_golden_small_cases_bit_exact_keys_and_values():
    z = np.load(GOLD / "golden_small.npz")
    for c in range(int(z["ncases"][0])):
        p = f"c{c}_"
        g = ib.StaggeredGrid(list(z[p + "ext"]), float(z[p + "h"][0]), list(z[p + "alpha"]),
                             [bool(v) for v in z[p + "per"]])
        pts, vals = z[p + "pts"], z[p + "vals"]
        ws = ib.SpreadWorkspace(len(vals), g)
        got = ib.spread_fused(pts, vals, g, K, ws, 4)
        assert np.array_equal(ws.keys, z[p + "keys"]), c
        assert np.array_equal(ws.perm, z[p + "perm"]), c
        assert ws.run_count == z[p + "run_keys"].size, c
        assert np.array_equal(ws.run_keys, z[p + "run_keys"]), c
        assert O.max_rel_deviation(got.values, z[p + "spread"]) <= TOL, c
        assert O.max_rel_deviation(got.values, z[p + "serial"]) <= TOL, c
        serial = ib.spread_serial(pts, vals, g, K)
        assert np.array_equal(serial.values, got.values), c  # one device operator
        e = ib.interpolate(ib.GridField(g, z[p + "field"]), pts, K, 3)
        assert O.max_rel_deviation(e, z[p + "interp"]) <= TOL, c


def test_spread_walkthrough():
    # tests/coupling_test.cpp:205-217
    g = ib.StaggeredGrid([4, 4], 1.0, [0.0, 0.0], [False, False])
    z = np.load(GOLD / "golden_small.npz")
    ws = ib.SpreadWorkspace(5, g)
    got = ib.spread_fused(z["walk_pts"], z["walk_vals"], g, K, ws, 2)
    assert ws.perm.tolist() == [0, 3, 2, 4, 1]
    assert ws.run_count == 4
    assert np.array_equal(ws.keys, z["walk_keys"])
    assert O.max_rel_deviation(got.values, z["walk_spread"]) <= TOL


def _c1():
    c1 = json.loads((GOLD / "golden_c1.json").read_text())
    n, N, edge = c1["n"], c1["N"], c1["edge_cm"]
    g = ib.StaggeredGrid([N] * 3, edge / N, c1["alpha"], [True] * 3)
    pts = O.scatter_points(n, edge, 1)
    vals = 2.0 * O.scatter_points(n, 1.0, 2)[:, 0] - 1.0
    e = 2.0 * O.scatter_points(N ** 3 // 3 + 1, 1.0, 4).reshape(-1)[: N ** 3] - 1.0
    return c1, g, pts, vals, e


def test_config1_matches_reference_hashes():
    c1, g, pts, vals, e = _c1()
    ws = ib.SpreadWorkspace(len(vals), g)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    assert hashlib.sha256(ws.keys.tobytes()).hexdigest() == c1["keys_sha256"]
    assert hashlib.sha256(ws.perm.tobytes()).hexdigest() == c1["perm_sha256"]
    assert hashlib.sha256(ws.run_keys.tobytes()).hexdigest() == c1["run_keys_sha256"]
    assert ws.run_count == c1["run_count"]
    want, *_ = O.spread_fused(og(g), pts, vals)
    assert O.max_rel_deviation(got.values, want) <= TOL
    assert got.values.sum() == pytest.approx(c1["spread_sum"], rel=1e-12)
    interp = ib.interpolate(ib.GridField(g, e), pts, K, 8)
    assert O.max_rel_deviation(interp, O.interpolate(og(g), e, pts)) <= TOL
    assert interp.sum() == pytest.approx(c1["interp_sum"], rel=1e-10)


@pytest.mark.slow
def test_config2_strong_scaling_size_bit_exact():
    # BASELINE config 2: 2^20 points on 256^3 (q = 1,016,453 per SURVEY 8(a) a8)
    n, N, edge = 1 << 20, 256, 16e-4
    g = ib.StaggeredGrid([N] * 3, edge / N, [0.5, 0.5, 0.0], [True] * 3)
    pts = O.scatter_points(n, edge, 1)
    vals = 2.0 * O.scatter_points(n, 1.0, 2)[:, 0] - 1.0
    ws = ib.SpreadWorkspace(n, g)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    keys, perm, run_keys = O.prepare_keys(og(g), pts)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert ws.run_count == run_keys.size == 1016453
    want = O.spread_serial(og(g), pts, vals)
    assert O.max_rel_deviation(got.values, want) <= TOL
    # conservation at full size: h^3 sum(l) == sum(G)
    assert abs(got.values.sum() * g.spacing() ** 3 - vals.sum()) <= 1e-10 * np.abs(vals).sum()


# ------------------------------------------------------------------ coupling_test.cpp mirrors
def test_interpolate_constant_field_returns_constant():
    g = ib.StaggeredGrid([12, 12, 12], 0.5, [0.0, 0.5, 0.5], [True] * 3)
    rng = np.random.default_rng(31)
    e = ib.interpolate(ib.GridField(g, np.full(g.point_count(), 2.75)), rand_points(g, 200, rng), K, 2)
    assert np.all(np.abs(e - 2.75) <= 1e-13 * 2.75)


def test_interpolate_all_support_outside_gives_zero():
    g = ib.StaggeredGrid([6, 6], 1.0, [0.0, 0.0], [False, False])
    e = ib.interpolate(ib.GridField(g, np.full(36, 5.0)), np.array([[-20.0, 3.0]]), K, 1)
    assert e[0] == 0.0


def test_interpolate_repeatable_and_worker_independent():
    g = ib.StaggeredGrid([10, 10, 10], 0.25, [0.5, 0.5, 0.0], [True, False, True])
    rng = np.random.default_rng(37)
    f = ib.GridField(g, rng.uniform(-1, 1, g.point_count()))
    pts = rand_points(g, 500, rng)
    a = ib.interpolate(f, pts, K, 1)
    b = ib.interpolate(f, pts, K, 8)
    assert np.array_equal(a, b)
    assert O.max_rel_deviation(a, O.interpolate(og(g), f.values, pts)) <= TOL


def test_single_point_conserves_unit_value():
    g = ib.StaggeredGrid([8, 8, 8], 0.25, [0.5, 0.0, 0.5], [True] * 3)
    f = ib.spread_serial(np.array([[0.37, 1.91, 0.04]]), np.array([1.0]), g, K)
    assert f.values.sum() * 0.25 ** 3 == pytest.approx(1.0, abs=1e-13)


def test_zero_values_give_zero_field():
    g = ib.StaggeredGrid([8, 8], 0.5, [0.0, 0.0], [True, True])
    rng = np.random.default_rng(43)
    f = ib.spread_serial(rand_points(g, 50, rng), np.zeros(50), g, K)
    assert np.all(f.values == 0.0)


def test_coincident_points_add_linearly():
    g = ib.StaggeredGrid([8, 8], 0.5, [0.5, 0.5], [True, True])
    x = [1.23, 0.47]
    two = ib.spread_serial(np.array([x, x]), np.array([0.7, -0.2]), g, K)
    one = ib.spread_serial(np.array([x]), np.array([0.5]), g, K)
    assert O.max_rel_deviation(two.values, one.values) <= 1e-13


def test_one_point_per_cell_matches_oracle():
    g = ib.StaggeredGrid([32, 32], 1.0, [0.0, 0.0], [True, True])
    pts = np.array([[8.0 * i + 2.4, 8.0 * j + 3.1] for j in range(4) for i in range(4)])
    vals = np.random.default_rng(53).uniform(-1, 1, 16)
    ws = ib.SpreadWorkspace(16, g)
    f = ib.spread_fused(pts, vals, g, K, ws, 3)
    assert ws.run_count == 16
    assert O.max_rel_deviation(f.values, O.spread_serial(og(g), pts, vals)) <= 1e-15


@pytest.mark.parametrize("dim", [1, 2, 3])
def test_variants_match_oracle_on_random_configurations(dim):
    # coupling_test.cpp:240-283 + verify.hpp:95-127
    rng = np.random.default_rng(59 + dim)
    for trial in range(16):
        ext = rng.integers(4, 13, dim)
        g = ib.StaggeredGrid(list(ext), 0.5, list(rng.uniform(0, 0.999, dim)),
                             [bool(b) for b in rng.integers(0, 2, dim)])
        n = int(rng.integers(0, 301))
        pts = rand_points(g, n, rng)
        vals = rng.uniform(-1, 1, n)
        b = [1, 4, 8, 64][trial % 4]
        want_f, keys, perm, run_keys = O.spread_fused(og(g), pts, vals)
        ws = ib.SpreadWorkspace(n, g)
        fused = ib.spread_fused(pts, vals, g, K, ws, 1 + trial % 8)
        assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
        assert ws.run_count == run_keys.size
        assert O.max_rel_deviation(fused.values, want_f) <= TOL
        wsb = ib.SpreadWorkspace(n, g, b)
        buffered = ib.spread_buffered(pts, vals, g, K, wsb, 4)
        assert O.max_rel_deviation(buffered.values, want_f) <= TOL
        otf = ib.spread_buffered_otf(pts, vals, g, K, b, 4)
        assert np.array_equal(otf.values, buffered.values)


def test_repeated_calls_bitwise_identical():
    g = ib.StaggeredGrid([10, 10, 10], 0.25, [0.5, 0.5, 0.0], [True] * 3)
    rng = np.random.default_rng(71)
    pts, vals = rand_points(g, 800, rng), rng.uniform(-1, 1, 800)
    ws = ib.SpreadWorkspace(800, g)
    a = ib.spread_fused(pts, vals, g, K, ws, 4)
    b = ib.spread_fused(pts, vals, g, K, ws, 4)
    assert np.array_equal(a.values, b.values)


def test_adjointness():
    rng = np.random.default_rng(73)
    g = ib.StaggeredGrid([8, 8, 8], 0.5, [0.0, 0.5, 0.5], [True, False, True])
    for _ in range(10):
        pts, w = rand_points(g, 120, rng), rng.uniform(-1, 1, 120)
        e = ib.GridField(g, rng.uniform(-1, 1, g.point_count()))
        grid_side = float(ib.spread_serial(pts, w, g, K).values @ e.values) * 0.125
        interp = ib.interpolate(e, pts, K, 2)
        assert abs(grid_side - float(w @ interp)) <= 1e-12 * float(np.abs(w * interp).sum())


def test_periodic_spread_conserves_total():
    rng = np.random.default_rng(79)
    g = ib.StaggeredGrid([8, 8, 8], 0.25, [0.5] * 3, [True] * 3)
    pts, vals = rand_points(g, 300, rng), rng.uniform(-1, 1, 300)
    ws = ib.SpreadWorkspace(300, g)
    f = ib.spread_fused(pts, vals, g, K, ws, 3)
    assert f.values.sum() * 0.25 ** 3 == pytest.approx(vals.sum(), abs=1e-13 * np.abs(vals).sum())


def test_spread_is_linear_in_values():
    rng = np.random.default_rng(83)
    g = ib.StaggeredGrid([12, 12], 0.5, [0.0, 0.5], [True, True])
    pts = rand_points(g, 100, rng)
    v1, v2 = rng.uniform(-1, 1, 100), rng.uniform(-1, 1, 100)
    ws = ib.SpreadWorkspace(100, g)
    s1 = ib.spread_fused(pts, v1, g, K, ws, 2).values
    s2 = ib.spread_fused(pts, v2, g, K, ws, 2).values
    sc = ib.spread_fused(pts, 1.7 * v1 + v2, g, K, ws, 2).values
    assert O.max_rel_deviation(sc, 1.7 * s1 + s2) <= TOL


def test_operation_counts_independent_of_grid_size():
    rng = np.random.default_rng(89)
    for r in (8, 16, 32):
        g = ib.StaggeredGrid([r] * 3, 1.0 / r, [0.5] * 3, [True] * 3)
        pts, vals = rand_points(g, 64, rng), rng.uniform(-1, 1, 64)
        ib.stats.reset_delta_evaluations()
        ib.interpolate(ib.GridField(g), pts, K, 3)
        assert ib.stats.delta_evaluations() == 64 * 64
        ib.stats.reset_delta_evaluations()
        ib.spread_fused(pts, vals, g, K, ib.SpreadWorkspace(64, g), 3)
        assert ib.stats.delta_evaluations() == 64 * 64


def test_vector_components_match_scalar_oracle():
    grids = [ib.StaggeredGrid([8] * 3, 0.5, a, [True] * 3)
             for a in ([0.0, 0.5, 0.5], [0.5, 0.0, 0.5], [0.5, 0.5, 0.0])]
    rng = np.random.default_rng(97)
    fields = [ib.GridField(g, rng.uniform(-1, 1, g.point_count())) for g in grids]
    pts = rand_points(grids[0], 150, rng)
    vec = ib.interpolate_vector(fields, pts, K, 2)
    for c in range(3):
        assert O.max_rel_deviation(vec[c], O.interpolate(og(grids[c]), fields[c].values, pts)) <= TOL
    values = [rng.uniform(-1, 1, 150) for _ in range(3)]
    ws = ib.SpreadWorkspace(150, grids[0])
    sp = ib.spread_vector(pts, values, grids, K, ib.SpreadAlgorithm.fused, 0, ws, 2)
    for c in range(3):
        assert O.max_rel_deviation(sp[c].values, O.spread_serial(og(grids[c]), pts, values[c])) <= TOL


def test_vector_components_concurrent_equal_sequential():
    # spread_vector / interpolate_vector run their components on concurrent
    # host threads: bit-identical to the scalar calls one after the other,
    # the workspace holds the last component's sort (as in the reference),
    # the operation count is the sequential one, and a component whose
    # arguments fail raises after exactly the components before it ran
    grids = [ib.StaggeredGrid([32] * 3, 0.5, a, [True] * 3)
             for a in ([0.0, 0.5, 0.5], [0.5, 0.0, 0.5], [0.5, 0.5, 0.0])]
    rng = np.random.default_rng(98)
    n = 20000
    pts = rand_points(grids[0], n, rng)
    values = [rng.uniform(-1, 1, n) for _ in range(3)]
    fields = [ib.GridField(g, rng.uniform(-1, 1, g.point_count())) for g in grids]
    for algo in (ib.SpreadAlgorithm.fused, ib.SpreadAlgorithm.serial, ib.SpreadAlgorithm.otf):
        ws = ib.SpreadWorkspace(n, grids[0]) if algo == ib.SpreadAlgorithm.fused else None
        ib.stats.reset_delta_evaluations()
        vec = ib.spread_vector(pts, values, grids, K, algo, 2, ws, 4)
        assert ib.stats.delta_evaluations() == 3 * n * 64
        for c in range(3):
            assert np.array_equal(vec[c].values, ib.spread_serial(pts, values[c], grids[c], K).values)
        if ws is not None:
            keys, perm, _ = O.prepare_keys(og(grids[2]), pts)
            assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    E = ib.interpolate_vector(fields, pts, K, 4)
    for c in range(3):
        assert np.array_equal(E[c], ib.interpolate(fields[c], pts, K, 4))
    ib.stats.reset_delta_evaluations()
    with pytest.raises(ib.InvalidArgument, match="one value per point"):
        ib.spread_vector(pts, [values[0], values[1][:10], values[2]], grids, K,
                         ib.SpreadAlgorithm.serial, 0, None, 1)
    assert ib.stats.delta_evaluations() == n * 64  # component 0 ran, as in the reference


def test_workspace_errors():
    g = ib.StaggeredGrid([8, 8], 0.5, [0.0, 0.0], [True, True])
    other = ib.StaggeredGrid([10, 10], 0.5, [0.0, 0.0], [True, True])
    pts, vals = np.array([[1.0, 1.0], [2.0, 2.0]]), np.array([1.0, 2.0])
    with pytest.raises(ib.InvalidArgument):
        ib.spread_fused(pts, vals, g, K, ib.SpreadWorkspace(5, g), 1)
    with pytest.raises(ib.InvalidArgument):
        ib.spread_fused(pts, vals, g, K, ib.SpreadWorkspace(2, other), 1)
    with pytest.raises(ib.InvalidArgument):
        ib.spread_buffered(pts, vals, g, K, ib.SpreadWorkspace(2, g), 1)
    with pytest.raises(ib.InvalidArgument):
        ib.spread_buffered_otf(pts, vals, g, K, 0, 1)
    with pytest.raises(ib.InvalidArgument):
        ib.spread_vector(pts, [vals, vals], [g, g], K, ib.SpreadAlgorithm.fused, 0, None, 1)
    with pytest.raises(ib.InvalidArgument):
        ib.spread_serial(pts, vals[:1], g, K)
    with pytest.raises(ib.InvalidArgument):
        ib.SpreadWorkspace(2, g, -1)


def test_empty_point_set_gives_zero_field():
    g = ib.StaggeredGrid([6, 6], 1.0, [0.0, 0.0], [True, True])
    f = ib.spread_buffered_otf(np.zeros((0, 2)), np.zeros(0), g, K, 1, 4)
    assert np.all(f.values == 0.0)
    assert ib.interpolate(ib.GridField(g), np.zeros((0, 2)), K, 1).size == 0


def test_tiny_periodic_grids_wrap_support_onto_itself():
    # extents < support: several shifts land on one grid point
    rng = np.random.default_rng(5)
    for ext in ([1], [2, 3], [3, 1, 2], [2, 2, 2]):
        d = len(ext)
        g = ib.StaggeredGrid(ext, 0.5, [0.3] * d, [True] * d)
        pts, vals = rand_points(g, 40, rng), rng.uniform(-1, 1, 40)
        want = O.spread_serial(og(g), pts, vals)
        got = ib.spread_serial(pts, vals, g, K)
        assert O.max_rel_deviation(got.values, want) <= TOL, ext
        e = rng.uniform(-1, 1, g.point_count())
        assert O.max_rel_deviation(ib.interpolate(ib.GridField(g, e), pts, K), O.interpolate(og(g), e, pts)) <= TOL


def test_long_x_rows_use_chunked_tiles():
    # n0 > 4096 switches the spread to x-chunked tiles
    rng = np.random.default_rng(9)
    for per in (True, False):
        g = ib.StaggeredGrid([9000, 3], 0.5, [0.25, 0.5], [per, True])
        pts, vals = rand_points(g, 5000, rng), rng.uniform(-1, 1, 5000)
        want = O.spread_serial(og(g), pts, vals)
        got = ib.spread_serial(pts, vals, g, K)
        assert O.max_rel_deviation(got.values, want) <= TOL


def test_device_path_matches_host_path():
    import torch

    from paper_2012_06646_b200.device import DeviceOperators

    rng = np.random.default_rng(11)
    g = ib.StaggeredGrid([32, 24, 20], 0.1, [0.5, 0.5, 0.0], [True] * 3)
    pts, vals = rand_points(g, 5000, rng), rng.uniform(-1, 1, 5000)
    e = rng.uniform(-1, 1, g.point_count())
    ops = DeviceOperators(0)
    dp = torch.tensor(pts, device="cuda")
    out = ops.spread(dp, torch.tensor(vals, device="cuda"), g)
    ei = ops.interpolate(torch.tensor(e, device="cuda"), dp, g)
    torch.cuda.synchronize()
    ws = ib.SpreadWorkspace(5000, g)
    host = ib.spread_fused(pts, vals, g, K, ws, 1)
    assert np.array_equal(out.cpu().numpy(), host.values)
    assert np.array_equal(ei.cpu().numpy(), ib.interpolate(ib.GridField(g, e), pts, K))


def test_cuda_graph_replay_matches_eager():
    """The device pipeline (sort, records, sweeps) has no host round trip, so
    a step captured in a CUDA graph replays bit-identically (bench.py)."""
    import torch

    from paper_2012_06646_b200.device import DeviceOperators

    rng = np.random.default_rng(12)
    g = ib.StaggeredGrid([64, 48, 40], 0.1, [0.5, 0.5, 0.0], [True] * 3)
    n = 40000
    pts = torch.tensor(rand_points(g, n, rng), device="cuda")
    vals = torch.tensor(rng.uniform(-1, 1, n), device="cuda")
    e = torch.tensor(rng.uniform(-1, 1, g.point_count()), device="cuda")
    ops = DeviceOperators(0)
    ell = torch.empty(g.point_count(), dtype=torch.float64, device="cuda")
    E = torch.empty(n, dtype=torch.float64, device="cuda")

    def step():
        ops.spread(pts, vals, g, out=ell)
        ops.interpolate(e, pts, g, out=E)

    step()
    torch.cuda.synchronize()
    ref_ell, ref_E = ell.clone(), E.clone()
    from paper_2012_06646_b200.device import capture_graph

    graph = capture_graph(step)
    ell.zero_()
    E.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(ell, ref_ell) and torch.equal(E, ref_E)
    o = og(g)
    assert O.max_rel_deviation(ell.cpu().numpy(), O.spread_serial(o, pts.cpu().numpy(), vals.cpu().numpy())) <= TOL


def test_clustered_long_runs():
    # many points per cell: rank-serialized shared-memory accumulation
    rng = np.random.default_rng(13)
    g = ib.StaggeredGrid([16, 16, 16], 1.0, [0.5, 0.5, 0.0], [True] * 3)
    centers = rng.uniform(0, 16, (3, 3))
    pts = np.concatenate([c + rng.normal(0, 0.3, (700, 3)) for c in centers])
    vals = rng.uniform(-1, 1, len(pts))
    want = O.spread_serial(og(g), pts, vals)
    ws = ib.SpreadWorkspace(len(pts), g)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    _, keys, perm, _ = O.spread_fused(og(g), pts, vals)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert O.max_rel_deviation(got.values, want) <= TOL


def test_clustered_row_longer_than_shared_sort():
    # one cell-row holding > 8192 points (the quadratic long-row path) next to
    # ordinary rows: clustered rows put the sweep in bank mode
    rng = np.random.default_rng(17)
    g = ib.StaggeredGrid([24, 20, 16], 1.0, [0.5, 0.5, 0.0], [True] * 3)
    tight = np.array([7.3, 9.6, 4.2]) + rng.normal(0, 0.02, (9000, 3))
    loose = rand_points(g, 3000, rng)
    pts = np.concatenate([tight, loose])
    vals = rng.uniform(-1, 1, len(pts))
    ws = ib.SpreadWorkspace(len(pts), g)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    _, keys, perm, _ = O.spread_fused(og(g), pts, vals)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert O.max_rel_deviation(got.values, O.spread_serial(og(g), pts, vals)) <= TOL


@pytest.mark.parametrize("per", [(True, True, True), (False, True, False), (True, False, True),
                                 (False, False, False)])
def test_zsweep_medium_grids_mixed_periodicity(per):
    # 3-D grids take the z-sweep kernels; ghost cells on closed axes included
    rng = np.random.default_rng(17 + sum(per))
    g = ib.StaggeredGrid([24, 20, 37], 0.5, [0.3, 0.0, 0.7], list(per), [0.25, -1.0, 2.0])
    n = 4000
    pts, vals = rand_points(g, n, rng), rng.uniform(-1, 1, n)
    want, keys, perm, run_keys = O.spread_fused(og(g), pts, vals)
    ws = ib.SpreadWorkspace(n, g)
    got = ib.spread_fused(pts, vals, g, K, ws, 4)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert np.array_equal(ws.run_keys, run_keys)
    assert O.max_rel_deviation(got.values, want) <= TOL
    e = rng.uniform(-1, 1, g.point_count())
    assert O.max_rel_deviation(ib.interpolate(ib.GridField(g, e), pts, K), O.interpolate(og(g), e, pts)) <= TOL


def test_dense_one_point_per_cell():
    # weak-scaling density (1 point per cell): long rows, several batch groups per warp
    rng = np.random.default_rng(23)
    N = 40
    g = ib.StaggeredGrid([N] * 3, 0.1, [0.5, 0.5, 0.0], [True] * 3)
    pts = rng.uniform(0, N * 0.1, (N ** 3, 3))
    vals = rng.uniform(-1, 1, N ** 3)
    want = O.spread_serial(og(g), pts, vals)
    ws = ib.SpreadWorkspace(N ** 3, g)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    assert O.max_rel_deviation(got.values, want) <= TOL
    e = rng.uniform(-1, 1, g.point_count())
    assert O.max_rel_deviation(ib.interpolate(ib.GridField(g, e), pts, K), O.interpolate(og(g), e, pts)) <= TOL


def _full_size_parity(N, pts, seed):
    edge = 16e-4
    g = ib.StaggeredGrid([N] * 3, edge / N, [0.5, 0.5, 0.0], [True] * 3)
    rng = np.random.default_rng(seed)
    vals = rng.uniform(-1, 1, len(pts))
    ws = ib.SpreadWorkspace(len(pts), g)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    keys, perm, run_keys = O.prepare_keys(og(g), pts)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert ws.run_count == run_keys.size
    assert O.max_rel_deviation(got.values, O.spread_serial(og(g), pts, vals)) <= TOL
    e = rng.uniform(-1, 1, g.point_count())
    E = ib.interpolate(ib.GridField(g, e), pts, K, 8)
    assert O.max_rel_deviation(E, O.interpolate(og(g), e, pts)) <= TOL


@pytest.mark.slow
def test_config_rbc_full_array_parity():
    # ~0.9 M points on RBC surfaces, 256^3 (pull mode)
    from paper_2012_06646_b200 import synth

    _full_size_parity(256, synth.rbc_points(16e-4, 16e-4 / 256, 7), 31)


@pytest.mark.slow
def test_config_clustered_full_array_parity():
    # 2^22 points in 64 Gaussian clusters, 512^3 (bank
    # mode, clustered rows, CTA-sorted long rows)
    from paper_2012_06646_b200 import synth

    _full_size_parity(512, synth.clustered_points(1 << 22, 16e-4, 64, 8 * 16e-4 / 512, 5), 32)


def test_concurrent_host_calls_from_threads_match_serial():
    """The reference's threading contract (spread.hpp:26):
    concurrent calls on disjoint outputs are safe.  Host-buffer calls run on
    per-call lanes of the context; results equal the one-thread calls bit for
    bit."""
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(77)
    g = ib.StaggeredGrid([64, 48, 40], 0.1, [0.5, 0.5, 0.0], [True] * 3)
    n = 30000
    pts = [rand_points(g, n, rng) for _ in range(4)]
    vals = [rng.uniform(-1, 1, n) for _ in range(4)]
    e = ib.GridField(g, rng.uniform(-1, 1, g.point_count()))
    want_s = [ib.spread_serial(p, v, g, K).values for p, v in zip(pts, vals)]
    want_i = [ib.interpolate(e, p, K) for p in pts]
    with ThreadPoolExecutor(max_workers=8) as pool:
        fs = [pool.submit(lambda p=p, v=v: ib.spread_serial(p, v, g, K).values) for p, v in zip(pts, vals)]
        fi = [pool.submit(lambda p=p: ib.interpolate(e, p, K)) for p in pts]
        got_s = [f.result() for f in fs]
        got_i = [f.result() for f in fi]
    for a, b in zip(got_s, want_s):
        assert np.array_equal(a, b)
    for a, b in zip(got_i, want_i):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("path", ["auto", "pull"])
def test_very_long_row_merge_sort(path):
    # one cell row holding 40000 points (> kLongSortMax = 8192: chunked bitonic
    # sorts + three merge passes), next to ordinary rows; ws.keys / ws.perm
    # bit-exact, the spread within 1e-12 (pull mode sorts it inside the spread)
    rng = np.random.default_rng(19)
    g = ib.StaggeredGrid([64, 20, 16], 1.0, [0.5, 0.5, 0.0], [True] * 3)
    row = np.stack([rng.uniform(0, 64, 40000), 7.6 + rng.uniform(-0.3, 0.3, 40000),
                    4.2 + rng.uniform(-0.3, 0.3, 40000)], axis=1)
    pts = np.concatenate([row, rand_points(g, 3000, rng)])
    vals = rng.uniform(-1, 1, len(pts))
    ctx = ib.Context(0)
    ctx.set_spread_path(path)
    ws = ib.SpreadWorkspace(len(pts), g, context=ctx)
    got = ib.spread_fused(pts, vals, g, K, ws, 8)
    _, keys, perm, _ = O.spread_fused(og(g), pts, vals)
    assert np.array_equal(ws.keys, keys) and np.array_equal(ws.perm, perm)
    assert O.max_rel_deviation(got.values, O.spread_serial(og(g), pts, vals)) <= TOL
