"""Device-resident MAC step loop (paper_2012_06646_b200/step.py) against the
reference's bench step (inc/bench/run.hpp:59-128) restated over the oracle."""
import numpy as np
import pytest

import oracle as O
from paper_2012_06646_b200 import step as S
from paper_2012_06646_b200 import synth

TOL = 1e-12


def test_step_config_defaults_match_reference():
    c = S.StepConfig()
    assert (c.refinement, c.point_count, c.domain_edge_um) == (64, 1 << 16, 16.0)
    assert (c.dt_us, c.shear_rate, c.spring_constant, c.seed) == (0.1, 1000.0, 0.01, 1)
    g = S.mac_grids(16, c.edge_cm)
    assert [list(x.staggerings) for x in g] == [[0.0, 0.5, 0.5], [0.5, 0.0, 0.5], [0.5, 0.5, 0.0]]


def _og(g):
    return O.make_grid(g.extents, g.spacing(), g.staggerings, g.periodic, g.origin)


def _reference_loop(cfg, steps):
    """run_benchmark's step, numpy + oracle operators (setup.hpp, run.hpp)."""
    L, dt = cfg.edge_cm, cfg.dt_s
    grids = [_og(g) for g in S.mac_grids(cfg.refinement, L)]
    N = cfg.refinement
    h = L / N
    y = h * (np.arange(N) + 0.5)
    u2 = np.broadcast_to((cfg.shear_rate * (y - 0.5 * L))[None, :, None], (N, N, N)).reshape(-1)
    vel = [np.zeros(N ** 3), np.zeros(N ** 3), np.ascontiguousarray(u2)]
    X = synth.scatter_points(cfg.point_count, L, cfg.seed).copy()
    X0 = X.copy()
    ell = None
    for _ in range(steps):
        u = np.stack([O.interpolate(g, vel[a], X) for a, g in enumerate(grids)])
        Xs = X + dt * u.T
        d = Xs - X0
        d -= L * np.round(d / L)
        F = -cfg.spring_constant * d
        ell = [O.spread_serial(g, Xs, F[:, a]) for a, g in enumerate(grids)]
        u2_ = np.stack([O.interpolate(g, vel[a], X) for a, g in enumerate(grids)])
        X = X + dt * u2_.T
    return X, ell


@pytest.mark.gpu
def test_mac_step_loop_matches_reference_step():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    # A shear rate large enough that points cross cells within the test.
    cfg = S.StepConfig(refinement=16, point_count=3000, dt_us=100.0)
    loop = S.MacStepLoop(cfg)
    for _ in range(4):
        loop.step()
    torch.cuda.synchronize()
    X_ref, ell_ref = _reference_loop(cfg, 4)
    X = loop.X.cpu().numpy()
    assert np.abs(X - X_ref).max() <= TOL * cfg.edge_cm
    assert np.abs(X - synth.scatter_points(cfg.point_count, cfg.edge_cm, cfg.seed)).max() > 0.1 * cfg.edge_cm / 16
    for a in range(3):
        got = loop.spread_result[a].cpu().numpy()
        if not np.any(ell_ref[a]):  # shear flow along z: no x / y tether forces
            assert not np.any(got)
        else:
            assert O.max_rel_deviation(got, ell_ref[a]) <= TOL


@pytest.mark.gpu
def test_mac_step_loop_graph_replay_matches_eager():
    """bench.py times the MAC step replayed from a CUDA graph: same state as
    the eager loop, bit for bit."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = S.StepConfig(refinement=16, point_count=2000, dt_us=100.0)
    eager = S.MacStepLoop(cfg)
    for _ in range(3):
        eager.step()
    torch.cuda.synchronize()
    loop = S.MacStepLoop(cfg)
    loop.step()  # warm-up (allocations, kernel attributes) ...
    torch.cuda.synchronize()
    loop.X.copy_(loop.anchors)  # ... then back to the initial state
    from paper_2012_06646_b200.device import capture_graph

    graph = capture_graph(loop.step)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(loop.X, eager.X)
    for a in range(3):
        assert torch.equal(loop.spread_result[a], eager.spread_result[a])


def test_fnv1a_and_csv_schema():
    # run.hpp:44-52 (FNV-1a 64: offset basis, prime) and report.hpp:16-18, 50-66
    import io

    assert S.fnv1a(b"") == 14695981039346656037
    assert S.fnv1a(b"a") == 0xAF63DC4C8601EC8C
    assert S.fnv1a(b"foobar") == 0x85944171F73967E8
    rep = S.TimingReport(S.StepConfig(refinement=32, point_count=1024, steps=2, seed=7),
                         interpolate_seconds=[1e-3, 3e-3, 2e-3, 2e-3], spread_seconds=[4e-3, 5e-3])
    buf = io.StringIO()
    S.write_csv([rep], buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == ("algorithm,refinement,n_points,workers,sweep_width,operation,calls,"
                        "mean_s,min_s,max_s,seed")
    assert lines[1] == "fused,32,1024,1,8,interpolate,4,2.000000000e-03,1.000000000e-03,3.000000000e-03,7"
    assert lines[2] == "fused,32,1024,1,8,spread,2,4.500000000e-03,4.000000000e-03,5.000000000e-03,7"


@pytest.mark.gpu
def test_binned_interpolation_equals_plain_interpolation():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2012_06646_b200 import ib
    from paper_2012_06646_b200.device import DeviceOperators

    rng = np.random.default_rng(5)
    ops = DeviceOperators(0)
    for ext, per in (([64, 48, 40], [True] * 3), ([30, 20, 12], [False, True, False]),
                     ([40, 24], [True, False])):
        g = ib.StaggeredGrid(ext, 0.5, [0.5] * len(ext), per)
        n = 20000
        pts = np.stack([rng.uniform(-0.5 * e, 1.2 * e, n) * 0.5 for e in ext], 1)
        dp = torch.tensor(pts, device="cuda")
        b = ops.bin_points(dp, g)
        for _ in range(2):  # several fields at one binning
            f = torch.tensor(rng.uniform(-1, 1, g.point_count()), device="cuda")
            want = ops.interpolate(f, dp, g)
            got = ops.interpolate_binned(f, b)
            torch.cuda.synchronize()
            assert torch.equal(got, want)
            assert O.max_rel_deviation(got.cpu().numpy(), O.interpolate(_og(g), f.cpu().numpy(), pts)) <= TOL


@pytest.mark.gpu
def test_run_benchmark_report_and_determinism():
    # verify.hpp check_determinism: same config and seed -> same positions and
    # fingerprint; two interpolation timings and one spread timing per step
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = S.StepConfig(refinement=16, point_count=1 << 10, steps=3, dt_us=50.0)
    a = S.run_benchmark(cfg)
    b = S.run_benchmark(cfg)
    assert len(a.interpolate_seconds) == 6 and len(a.spread_seconds) == 3
    assert a.physics_fingerprint == b.physics_fingerprint != 0
    assert np.array_equal(a.final_positions, b.final_positions)
    X_ref, _ = _reference_loop(cfg, 3)
    assert np.abs(a.final_positions - X_ref).max() <= TOL * cfg.edge_cm
