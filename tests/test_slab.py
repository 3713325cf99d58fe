"""Multi-rank z-slab decomposition (paper_2012_06646_b200/slab.py).

CPU (gloo, world size 2 and 3): the decomposition logic -- slab bounds, point
binning by home plane, ghost-plane sum after spreading, halo fill before
interpolating -- with the oracle as each rank's local operator, checked
against the single-grid oracle (max_rel_deviation <= 1e-12).

GPU (2 ranks on one device, gloo staging through host memory): the same with
the device slab operators (ibc_spread_slab_device / ibc_interpolate_slab_device,
global-coordinate cells), checked against the single-grid oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as O
from paper_2012_06646_b200 import ib
from paper_2012_06646_b200 import slab as S

TOL = 1e-12


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {
    # extents, spacing, staggering, periodic, n points
    "periodic": ((8, 6, 12), 0.5, (0.5, 0.25, 0.0), (True, True, True), 400),
    "closed_z": ((7, 6, 12), 0.5, (0.0, 0.5, 0.0), (True, False, False), 300),
    "planes2d": ((9, 10), 0.5, (0.25, 0.0), (True, True), 200),
}


def _inputs(case):
    ext, h, alpha, per, n = CASES[case]
    rng = np.random.default_rng(11)
    d = len(ext)
    pts = np.empty((n, d))
    for a in range(d):
        pts[:, a] = rng.uniform(0.0, ext[a] * h, n)  # wrapped, dyadic-exact slab shifts
    vals = rng.uniform(-1, 1, n)
    field = rng.uniform(-1, 1, int(np.prod(ext)))
    return ext, h, alpha, per, pts, vals, field


def _oracle_local_ops(dec, ext, h, alpha, per):
    """Each rank's local operator on CPU: the oracle on an ordinary grid equal
    to the slab's local grid (exact here: h = 0.5 and the shift is dyadic)."""
    lay = dec.lay
    lext = list(ext[:-1]) + [lay.local_planes]
    lper = list(per[:-1]) + [False]
    origin = [0.0] * len(ext)
    origin[-1] = (lay.z0 - 2) * h
    og = O.make_grid(lext, h, alpha, lper, origin)

    g_global = O.make_grid(list(ext), h, list(alpha), list(per))

    def shifted(points):
        # A point whose (unwrapped) home cell is n on a periodic slab axis is
        # homed in plane 0: move it down one period, as the device's
        # global-coordinate slab cells do (ibc_device.cuh cell_of_slab).
        p = points.numpy().copy()
        if per[-1]:
            cu = O.home_cells(g_global, p, wrap=False)[:, -1]
            p[:, -1] -= (cu // ext[-1]) * ext[-1] * h
        return p

    def spread(points, values):
        return torch.from_numpy(O.spread_serial(og, shifted(points), values.numpy()))

    def interp(field, points):
        return torch.from_numpy(O.interpolate(og, field.numpy(), shifted(points)))

    return spread, interp


def _cpu_worker(rank, world, port, case, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=world)
        ext, h, alpha, per, pts, vals, field = _inputs(case)
        grid = ib.StaggeredGrid(list(ext), h, list(alpha), list(per))
        dec = S.SlabDecomposition(grid, rank, world)
        dec._spread, dec._interp = _oracle_local_ops(dec, ext, h, alpha, per)
        og = O.make_grid(list(ext), h, list(alpha), list(per))
        planes = torch.from_numpy(O.home_cells(og, pts)[:, -1])
        mine = (S.owner_of_planes(planes, ext[-1], world) == rank).numpy()
        lay, P = dec.lay, dec.lay.plane
        # spread: owned planes == the single-grid oracle's planes [z0, z1)
        own = dec.spread(torch.from_numpy(pts[mine]), torch.from_numpy(vals[mine]))
        want = O.spread_serial(og, pts, vals)[lay.z0 * P:lay.z1 * P]
        dev = O.max_rel_deviation(own.numpy(), want)
        assert dev <= TOL, f"rank {rank} spread dev {dev}"
        # interpolate: owned planes of the field in, my points' values out
        owned = torch.from_numpy(field[lay.z0 * P:lay.z1 * P].copy())
        e = dec.interpolate(owned, torch.from_numpy(pts[mine]))
        want_e = O.interpolate(og, field, pts)[mine]
        dev = O.max_rel_deviation(e.numpy(), want_e)
        assert dev <= TOL, f"rank {rank} interp dev {dev}"
        dist.destroy_process_group()
    except BaseException as exc:  # pragma: no cover - reported to the parent
        errq.put(f"rank {rank}: {exc!r}")


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_slab_bounds_and_layout():
    assert S.slab_bounds(12, 2) == [0, 6, 12]
    assert S.slab_bounds(256, 3) == [0, 85, 170, 256]
    with pytest.raises(ValueError):
        S.slab_bounds(5, 3)
    g = ib.StaggeredGrid([8, 6, 12], 0.5, [0.5, 0.5, 0.0], [True] * 3)
    lay = S.layout(g, 1, 2)
    assert (lay.z0, lay.z1, lay.plane, lay.local_planes, lay.z_first) == (6, 12, 48, 9, 4)
    loc = S.local_grid(g, lay)
    assert loc.extents == (8, 6, 9) and loc.periodic == (True, True, False)
    assert loc.origin == g.origin  # the slab shift travels in ibc_slab, not the origin
    planes = torch.tensor([0, 5, 6, 11, 12], dtype=torch.int32)
    assert S.owner_of_planes(planes, 12, 2).tolist() == [0, 0, 1, 1, 1]


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_matches_single_grid_oracle(case, world):
    _spawn(_cpu_worker, world, case)


def _gpu_worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ext, h, alpha, per, n = (32, 24, 40), 0.5, (0.5, 0.5, 0.0), (True, True, True), 6000
        rng = np.random.default_rng(5)
        pts = np.stack([rng.uniform(-2.0, ext[a] * h + 2.0, n) for a in range(3)], axis=1)
        vals = rng.uniform(-1, 1, n)
        field = rng.uniform(-1, 1, int(np.prod(ext)))
        grid = ib.StaggeredGrid(list(ext), h, list(alpha), list(per))
        og = O.make_grid(list(ext), h, list(alpha), list(per))
        dec = S.SlabDecomposition(grid, rank, world)
        X = torch.tensor(pts, device="cuda")
        planes = S.home_planes(grid, X)
        assert np.array_equal(planes.cpu().numpy(), O.home_cells(og, pts)[:, -1])
        mine = (S.owner_of_planes(planes, ext[-1], world) == rank)
        lay, P = dec.lay, dec.lay.plane
        own = dec.spread(X[mine].contiguous(), torch.tensor(vals, device="cuda")[mine].contiguous())
        want = O.spread_serial(og, pts, vals)[lay.z0 * P:lay.z1 * P]
        dev = O.max_rel_deviation(own.cpu().numpy(), want)
        assert dev <= TOL, f"rank {rank} spread dev {dev}"
        owned = torch.tensor(field[lay.z0 * P:lay.z1 * P], device="cuda")
        e = dec.interpolate(owned, X[mine].contiguous())
        dev = O.max_rel_deviation(e.cpu().numpy(), O.interpolate(og, field, pts)[mine.cpu().numpy()])
        assert dev <= TOL, f"rank {rank} interp dev {dev}"
        torch.cuda.synchronize()
        dist.destroy_process_group()
    except BaseException as exc:  # pragma: no cover
        errq.put(f"rank {rank}: {exc!r}")


@pytest.mark.gpu
def test_device_slab_decomposition_two_ranks_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _spawn(_gpu_worker, 2)


@pytest.mark.gpu
def test_cpp_multi_rank_peer_exchange():
    """tests/cpp/slab_test.cpp: R = 1..4 ranks (host threads, own contexts and
    streams) spread, ghost-sum over peer memory, halo-fill and interpolate
    through the C ABI; matches the single-grid operators within 1e-12."""
    import subprocess

    from paper_2012_06646_b200 import _build

    exe = _build.build_slab_test()
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "slab ok" in out.stdout


def _peer_case(R, periodic, seed):
    ext, h = (32, 24, 8 * R), 0.5
    rng = np.random.default_rng(seed)
    n = 5000
    zlo, zhi = ((-ext[2] * h, 2 * ext[2] * h) if periodic else (2.0 * h, (ext[2] - 2) * h))
    pts = np.stack([rng.uniform(0, ext[0] * h, n), rng.uniform(0, ext[1] * h, n),
                    rng.uniform(zlo, zhi, n)], axis=1)
    vals = rng.uniform(-1, 1, n)
    field = rng.uniform(-1, 1, int(np.prod(ext)))
    per = (True, True, periodic)
    grid = ib.StaggeredGrid(list(ext), h, [0.5, 0.5, 0.0], list(per))
    og = O.make_grid(list(ext), h, [0.5, 0.5, 0.0], list(per))
    return grid, og, pts, vals, field


@pytest.mark.gpu
@pytest.mark.parametrize("R,periodic", [(1, True), (2, True), (2, False), (3, True), (3, False)])
def test_peer_transport_in_process(R, periodic):
    """PeerSlab with ranks in one process (own contexts and streams, peers
    wired directly): spread + peer ghost sum, halo fill + gather, vs the
    single-grid oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2012_06646_b200.device import DeviceOperators

    grid, og, pts, vals, field = _peer_case(R, periodic, 40 + R)
    X = torch.tensor(pts, device="cuda")
    planes = S.home_planes(grid, X)
    owner = S.owner_of_planes(planes, grid.extents[-1], R)
    decs, streams, parts = [], [], []
    for r in range(R):
        ops = DeviceOperators(0)
        decs.append(S.SlabDecomposition(grid, r, R, ops=ops))
        streams.append(torch.cuda.Stream())
        m = owner == r
        parts.append((m.cpu().numpy(), X[m].contiguous(),
                      torch.tensor(vals, device="cuda")[m].contiguous()))
    for r in range(R):  # warm-up: size every context's scratch before any handshake
        with torch.cuda.stream(streams[r]):
            decs[r]._device_spread(parts[r][1], parts[r][2])
            decs[r]._device_interpolate(torch.zeros(decs[r].local.point_count(), dtype=torch.float64,
                                                    device="cuda"), parts[r][1])
    torch.cuda.synchronize()
    slabs = []
    for d in decs:
        d.peer_slab = S.PeerSlab(d, d._device_ops())
        slabs.append(d.peer_slab)
    for d in decs:
        d.use_peer_transport(peers=slabs)
    owned, E = [], []
    for r in range(R):
        with torch.cuda.stream(streams[r]):
            owned.append(decs[r].spread(parts[r][1], parts[r][2]))
    for r in range(R):
        lay = decs[r].lay
        with torch.cuda.stream(streams[r]):
            own_f = torch.tensor(field[lay.z0 * lay.plane:lay.z1 * lay.plane], device="cuda")
            E.append(decs[r].interpolate(own_f, parts[r][1]))
    torch.cuda.synchronize()
    want = O.spread_serial(og, pts, vals)
    want_e = O.interpolate(og, field, pts)
    for r in range(R):
        lay = decs[r].lay
        assert not slabs[r].timed_out()
        dev = O.max_rel_deviation(owned[r].cpu().numpy(), want[lay.z0 * lay.plane:lay.z1 * lay.plane])
        assert dev <= TOL, (r, dev)
        assert O.max_rel_deviation(E[r].cpu().numpy(), want_e[parts[r][0]]) <= TOL
    for s_ in slabs:
        s_.close()


def _peer_worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        grid, og, pts, vals, field = _peer_case(world, True, 77)
        dec = S.SlabDecomposition(grid, rank, world)
        X = torch.tensor(pts, device="cuda")
        mine = S.owner_of_planes(S.home_planes(grid, X), grid.extents[-1], world) == rank
        xm, vm = X[mine].contiguous(), torch.tensor(vals, device="cuda")[mine].contiguous()
        dec._device_spread(xm, vm)  # warm-up before any handshake
        dec._device_interpolate(torch.zeros(dec.local.point_count(), dtype=torch.float64,
                                            device="cuda"), xm)
        torch.cuda.synchronize()
        dist.barrier()
        dec.use_peer_transport()  # CUDA IPC handles swapped over the gloo group
        dist.barrier()
        lay = dec.lay
        own = dec.spread(xm, vm)
        e = dec.interpolate(torch.tensor(field[lay.z0 * lay.plane:lay.z1 * lay.plane], device="cuda"), xm)
        torch.cuda.synchronize()
        assert not dec.peer.timed_out(), "handshake timed out"
        dev = O.max_rel_deviation(own.cpu().numpy(),
                                  O.spread_serial(og, pts, vals)[lay.z0 * lay.plane:lay.z1 * lay.plane])
        assert dev <= TOL, f"rank {rank} spread dev {dev}"
        dev = O.max_rel_deviation(e.cpu().numpy(), O.interpolate(og, field, pts)[mine.cpu().numpy()])
        assert dev <= TOL, f"rank {rank} interp dev {dev}"
        dist.barrier()
        dec.peer.close()
        dist.destroy_process_group()
    except BaseException as exc:  # pragma: no cover
        errq.put(f"rank {rank}: {exc!r}")


@pytest.mark.gpu
def test_peer_transport_two_processes_ipc():
    """Two processes, CUDA IPC peer pointers (the multi-GPU setup, here on
    one device)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _spawn(_peer_worker, 2)


def _migrate_worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist

        dist.init_process_group("gloo", rank=rank, world_size=world)
        ext, h = (8, 6, 12 * world), 0.5
        grid = ib.StaggeredGrid(list(ext), h, [0.5, 0.5, 0.0], [True] * 3)
        og = O.make_grid(list(ext), h, [0.5, 0.5, 0.0], [1, 1, 1])
        rng = np.random.default_rng(100)
        n = 3000
        pts = np.stack([rng.uniform(0, ext[a] * h, n) for a in range(3)], axis=1)
        moved = pts + rng.uniform(-1.5 * h, 1.5 * h, pts.shape)  # up to 1.5 cells per step
        ids = np.arange(n, dtype=np.float64)
        dec = S.SlabDecomposition(grid, rank, world)
        lay = dec.lay
        owner0 = S.owner_of_planes(torch.tensor(O.home_cells(og, pts)[:, 2]), ext[2], world)
        mine = (owner0 == rank).numpy()
        # this rank's points (old slab), at their new positions
        X = torch.tensor(moved[mine])
        planes = torch.tensor(O.home_cells(og, moved[mine])[:, 2])
        Xn, idn = dec.migrate(X, torch.tensor(ids[mine]), planes=planes)
        owner1 = S.owner_of_planes(torch.tensor(O.home_cells(og, moved)[:, 2]), ext[2], world).numpy()
        want = set(np.nonzero(owner1 == rank)[0].tolist())
        got = idn.numpy().astype(np.int64)
        assert sorted(got.tolist()) == sorted(want), f"rank {rank}: wrong set after migration"
        assert np.array_equal(Xn.numpy(), moved[got]), f"rank {rank}: rows scrambled"
        # the staying points first, in their order
        stay = [i for i in np.nonzero(mine)[0] if owner1[i] == rank]
        assert got[:len(stay)].tolist() == stay
        dist.destroy_process_group()
    except BaseException as exc:  # pragma: no cover
        errq.put(f"rank {rank}: {exc!r}")


@pytest.mark.parametrize("world", [2, 3])
def test_point_migration_between_neighbour_slabs(world):
    _spawn(_migrate_worker, world)
