"""Multi-GPU z-slab decomposition of the spread / interpolate path.

The reference runs on one shared-memory node (parallel.hpp:25-36); the paper
defers multi-device runs.  Here the grid's last axis (the slowest
in the colex layout, grid.hpp:136-151, so a slab is one contiguous range of a
GridField) is split into contiguous slabs, one per rank.  A rank owns home
planes [z0, z1) and the Lagrangian points homed there; it works on a LOCAL
grid of planes [z0 - 2, z1 + 1) (``ibc_slab``, include/ibcuda.h): cells are
computed in global coordinates, so keys and weights are those of the single
grid.

* spread: local spread into the z1 - z0 + 3 planes, then a **ghost-plane sum**:
  planes z0-2, z0-1 go to the rank below, plane z1 to the rank above, and each
  rank adds what it receives into the planes it owns;
* interpolate: a **halo fill** -- the two planes below the slab from the rank
  below, one plane above from the rank above -- then a local gather.

These two exchanges are the only communication on the path.  Two transports:

* ``"peer"`` (``PeerSlab``, the GPU default): the C ABI's peer-memory
  exchange -- each rank's local slab and signal block are shared with its
  ring neighbours through CUDA IPC handles (swapped once over the process
  group), and ``ibc_slab_ghost_sum_device`` / ``ibc_slab_halo_fill_device``
  pull the neighbours' planes over NVLink with device-side handshakes: no
  NCCL, no host synchronisation, the whole step capturable in one CUDA graph;
* ``"collective"``: torch.distributed send/recv between ring neighbours (NCCL
  batch_isend_irecv; a ``gloo`` group stages through host memory, which is
  what the CPU tests use).  On a closed (non-periodic) axis the outer ghost
planes fall off the grid, exactly like the reference's dropped out-of-grid
targets, and the outer halos are zero.

The local operators are injectable (``local_spread`` / ``local_interpolate``)
so the decomposition logic can be checked on CPU against the oracle; by
default they are the device operators of ``device.py``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _capi
from ._capi import check, load
from .ib import StaggeredGrid


@dataclass
class SlabLayout:
    """Where one rank's slab sits in the global grid."""

    rank: int
    world: int
    nz: int          # global extent of the last axis
    z0: int          # first owned plane
    z1: int          # one past the last owned plane
    plane: int       # values per plane (prod of the other extents)
    periodic: bool   # global periodicity of the last axis

    @property
    def nloc(self) -> int:
        return self.z1 - self.z0

    @property
    def local_planes(self) -> int:
        return self.nloc + 3

    @property
    def z_first(self) -> int:
        return self.z0 - 2


def slab_bounds(nz: int, world: int) -> list[int]:
    """Balanced contiguous split of nz planes over `world` ranks."""
    if world < 1 or nz < 2 * world:
        raise ValueError(f"cannot split {nz} planes over {world} ranks (need >= 2 each)")
    return [nz * r // world for r in range(world + 1)]


def layout(grid: StaggeredGrid, rank: int, world: int) -> SlabLayout:
    ext = list(grid.extents)
    b = slab_bounds(ext[-1], world)
    plane = 1
    for e in ext[:-1]:
        plane *= e
    return SlabLayout(rank, world, ext[-1], b[rank], b[rank + 1], plane, grid.is_periodic(grid.dim - 1))


def local_grid(grid: StaggeredGrid, lay: SlabLayout) -> StaggeredGrid:
    """The rank's local grid: planes [z0 - 2, z1 + 1), closed along the slab
    axis, same origin (the slab shift travels in ibc_slab, not in the origin)."""
    ext = list(grid.extents)
    ext[-1] = lay.local_planes
    per = list(grid.periodic)
    per[-1] = False
    return StaggeredGrid(ext, grid.spacing(), list(grid.staggerings), per, list(grid.origin))


def c_slab(lay: SlabLayout) -> _capi.IbcSlab:
    s = _capi.IbcSlab()
    s.z_first = lay.z_first
    s.nz_global = lay.nz
    s.periodic_global = int(lay.periodic)
    return s


class SlabDecomposition:
    """One rank's share of a z-slab decomposed spread / interpolate.

    Arrays are torch tensors (CUDA for the device operators; any device for
    injected local operators).  ``group`` is a torch.distributed process group
    (None = default group); with world == 1 the exchanges are local copies.
    """

    def __init__(self, grid: StaggeredGrid, rank: int, world: int, group=None,
                 local_spread=None, local_interpolate=None, ops=None):
        self.grid = grid
        self.lay = layout(grid, rank, world)
        self.local = local_grid(grid, self.lay)
        self.group = group
        self._ops = ops
        self._spread = local_spread or self._device_spread
        self._interp = local_interpolate or self._device_interpolate
        self.peer = None  # PeerSlab once use_peer_transport() is called

    # ---------------------------------------------------------- neighbours
    @property
    def down(self) -> int:
        return (self.lay.rank - 1) % self.lay.world

    @property
    def up(self) -> int:
        return (self.lay.rank + 1) % self.lay.world

    def _has_down(self) -> bool:
        return self.lay.periodic or self.lay.rank > 0

    def _has_up(self) -> bool:
        return self.lay.periodic or self.lay.rank < self.lay.world - 1

    def _exchange(self, send_down, send_up, recv_from_up_shape, recv_from_down_shape):
        """send_down -> rank below, send_up -> rank above; returns (from_up, from_down).

        Every rank posts the same four operations in the same order, so the
        two messages between a pair of ranks (world == 2: down == up) match in
        order."""
        import torch
        import torch.distributed as dist

        lay = self.lay
        like = send_down if send_down is not None else send_up
        if lay.world == 1:  # periodic ring of one: the neighbour is this rank
            return (send_down.clone() if self._has_up() else None,
                    send_up.clone() if self._has_down() else None)
        staged = dist.get_backend(self.group) != "nccl" and like.is_cuda
        dev = like.device

        def wire(t):
            return t.cpu().contiguous() if staged else t.contiguous()

        ops, from_up, from_down = [], None, None
        if self._has_down():
            ops.append(dist.P2POp(dist.isend, wire(send_down), self.down, self.group, tag=1))
        if self._has_up():
            ops.append(dist.P2POp(dist.isend, wire(send_up), self.up, self.group, tag=2))
        if self._has_up():
            from_up = torch.empty(recv_from_up_shape, dtype=like.dtype,
                                  device="cpu" if staged else dev)
            ops.append(dist.P2POp(dist.irecv, from_up, self.up, self.group, tag=1))
        if self._has_down():
            from_down = torch.empty(recv_from_down_shape, dtype=like.dtype,
                                    device="cpu" if staged else dev)
            ops.append(dist.P2POp(dist.irecv, from_down, self.down, self.group, tag=2))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if staged:
            from_up = from_up.to(dev) if from_up is not None else None
            from_down = from_down.to(dev) if from_down is not None else None
        return from_up, from_down

    # ------------------------------------------------------------- spread
    def ghost_sum(self, local_out):
        """Local spread output (local_planes x plane) -> the owned slab
        (nloc x plane): ghost planes to their owners, received ghosts added."""
        lay, P = self.lay, self.lay.plane
        L = local_out.view(lay.local_planes, P)
        from_up, from_down = self._exchange(L[0:2], L[lay.nloc + 2:lay.nloc + 3], (2, P), (1, P))
        own = L[2:lay.nloc + 2]
        if from_up is not None:    # the rank above's planes z1-2, z1-1
            own[lay.nloc - 2:lay.nloc] += from_up
        if from_down is not None:  # the rank below's plane z0
            own[0:1] += from_down
        return own.reshape(-1)

    def spread(self, points, values, out=None):
        """Points homed in this slab -> this rank's owned planes of the field."""
        if self.peer is not None:
            self._device_spread(points, values, out=self.peer.spread_buf)
            return self.peer.ghost_sum()
        return self.ghost_sum(self._spread(points, values))

    # -------------------------------------------------------- interpolate
    def halo_fill(self, owned, out=None):
        """Owned planes (nloc x plane) -> local field with halos (local_planes x plane)."""
        import torch

        lay, P = self.lay, self.lay.plane
        O = owned.view(lay.nloc, P)
        from_up, from_down = self._exchange(O[0:1], O[lay.nloc - 2:lay.nloc], (1, P), (2, P))
        if out is None:
            L = torch.zeros((lay.local_planes, P), dtype=owned.dtype, device=owned.device)
        else:
            L = out.view(lay.local_planes, P)
            if from_down is None:
                L[0:2].zero_()
            if from_up is None:
                L[lay.nloc + 2].zero_()
        L[2:lay.nloc + 2] = O
        if from_down is not None:  # planes z0-2, z0-1
            L[0:2] = from_down
        if from_up is not None:    # plane z1
            L[lay.nloc + 2] = from_up[0]
        return L.reshape(-1)

    def interpolate(self, owned_field, points, out=None):
        if self.peer is not None:
            dst = self.peer.owned_field
            if owned_field is not None and owned_field.data_ptr() != dst.data_ptr():
                dst.copy_(owned_field.reshape(-1))
            return self._device_interpolate(self.peer.halo_fill(), points, out=out)
        return self._interp(self.halo_fill(owned_field), points)

    def use_peer_transport(self, group=None, peers=None) -> "PeerSlab":
        """Switch this rank to the peer-memory exchange (PeerSlab): IPC over
        `group`, or the in-process `peers` list (set each rank's
        `.peer_slab` first, then call with peers=[...] on every rank)."""
        ps = self.peer_slab if getattr(self, "peer_slab", None) else PeerSlab(self, self._device_ops())
        self.peer_slab = ps
        if peers is not None:
            ps.connect_local(peers)
        else:
            ps.connect_ipc(group)
        self.peer = ps
        return ps

    # ---------------------------------------------------------- migration
    def migrate(self, points, *payloads, planes=None):
        """Per-step point migration between ring neighbours (SURVEY 2 K7,
        8(e)): points whose home plane left [z0, z1) go to the rank that owns
        it now -- a neighbour, since IB points move far less than a cell per
        step.  `planes`: the points' wrapped home planes on the
        global grid (default: `home_planes` on the device; injectable for CPU
        checks).  Returns (points, *payloads) of this rank after the move:
        the staying points in their order, then those from the rank below,
        then those from the rank above.  Counts go first, then the packed
        rows, over the same neighbour send/recv as the exchanges."""
        import torch

        lay = self.lay
        if planes is None:
            planes = home_planes(self.grid, points, self._device_ops())
        owner = owner_of_planes(planes.to(torch.int64), lay.nz, lay.world)
        stay = owner == lay.rank
        to_down = (owner == self.down) & ~stay
        to_up = (owner == self.up) & ~stay & ~to_down
        if bool((~(stay | to_down | to_up)).any()):
            raise ValueError("a point moved past a neighbouring slab in one step")
        cols = [points.reshape(points.shape[0], -1)] + [p.reshape(p.shape[0], -1) for p in payloads]
        widths = [c.shape[1] for c in cols]
        rows = torch.cat([c.to(torch.float64) for c in cols], dim=1)
        send_down, send_up = rows[to_down], rows[to_up]
        cnt_from_up, cnt_from_down = self._exchange(
            torch.tensor([send_down.shape[0]], dtype=torch.float64, device=rows.device),
            torch.tensor([send_up.shape[0]], dtype=torch.float64, device=rows.device), (1,), (1,))
        W = rows.shape[1]
        n_up = int(cnt_from_up.item()) if cnt_from_up is not None else 0
        n_down = int(cnt_from_down.item()) if cnt_from_down is not None else 0
        # Empty messages still travel (every rank posts the same operations).
        pad = lambda t: t if t.shape[0] else torch.zeros((1, W), dtype=t.dtype, device=t.device)
        from_up, from_down = self._exchange(pad(send_down), pad(send_up), (max(n_up, 1), W),
                                            (max(n_down, 1), W))
        parts = [rows[stay]]
        if from_down is not None and n_down:
            parts.append(from_down[:n_down])
        if from_up is not None and n_up:
            parts.append(from_up[:n_up])
        new = torch.cat(parts, dim=0)
        out, c0 = [], 0
        for c, w in zip(cols, widths):
            out.append(new[:, c0:c0 + w].to(c.dtype).reshape((-1,) + tuple(c.shape[1:]))
                       if w > 1 else new[:, c0].to(c.dtype))
            c0 += w
        out[0] = out[0].reshape(-1, points.shape[1]).contiguous()
        return tuple(o.contiguous() for o in out)

    # ---------------------------------------------------- device operators
    def _device_ops(self):
        if self._ops is None:
            import torch

            from .device import DeviceOperators

            self._ops = DeviceOperators(torch.cuda.current_device())
        return self._ops

    def _device_spread(self, points, values, out=None):
        import torch

        from .device import _ptr, _require

        ops = self._device_ops()
        n = points.shape[0]
        _require(points, "points", n * self.grid.dim)
        _require(values, "values", n)
        if out is None:
            out = torch.empty(self.local.point_count(), dtype=torch.float64, device=points.device)
        ws = ops.workspace(n, self.local)
        ops._sync_stream()
        slab = c_slab(self.lay)
        check(load().ibc_spread_slab_device(ops.context.handle, C.byref(self.local.c_grid),
                                            C.byref(slab), _capi.IBC_KERNEL_COSINE4,
                                            _ptr(points), _ptr(values), n, ws.handle, _ptr(out)))
        return out

    def _device_interpolate(self, field_local, points, out=None):
        import torch

        from .device import _ptr, _require

        ops = self._device_ops()
        n = points.shape[0]
        _require(field_local, "field", self.local.point_count())
        _require(points, "points", n * self.grid.dim)
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=points.device)
        ops._sync_stream()
        slab = c_slab(self.lay)
        check(load().ibc_interpolate_slab_device(ops.context.handle, C.byref(self.local.c_grid),
                                                 C.byref(slab), _capi.IBC_KERNEL_COSINE4,
                                                 _ptr(field_local), _ptr(points), n, _ptr(out)))
        return out


def home_planes(grid: StaggeredGrid, points, ops=None):
    """Wrapped home cell along the last axis of every point (device): the
    slab-binning key, bit-identical to the reference's cell_index + wrap."""
    import torch

    from .device import DeviceOperators, _ptr, _require

    ops = ops or DeviceOperators(torch.cuda.current_device())
    n = points.shape[0]
    _require(points, "points", n * grid.dim)
    out = torch.empty(n, dtype=torch.int32, device=points.device)
    ops._sync_stream()
    check(load().ibc_home_planes_device(ops.context.handle, C.byref(grid.c_grid),
                                        _capi.IBC_KERNEL_COSINE4, _ptr(points), n, _ptr(out)))
    return out


def owner_of_planes(planes, nz: int, world: int):
    """Rank owning each home plane (torch int tensor in, int64 out)."""
    import torch

    b = torch.tensor(slab_bounds(nz, world)[1:-1], dtype=planes.dtype, device=planes.device)
    return torch.bucketize(planes.contiguous(), b, right=True)


# ---------------------------------------------------------------- peer transport
class _DeviceArray:
    """__cuda_array_interface__ view of library-allocated device memory."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class PeerSlab:
    """This rank's slab buffers, shared with its ring neighbours over peer
    memory (include/ibcuda.h ibc_slab_link): `spread_buf` (the local spread
    output, ghost-summed in place) and `field_buf` (the local interpolation
    field, halo-filled in place), both nloc + 3 planes, plus a signal block.

    Wire the neighbours with `connect_ipc(group)` (one process per rank:
    CUDA IPC handles swapped over the process group) or `connect_local(peers)`
    (ranks in one process).  Every rank then calls `ghost_sum()` /
    `halo_fill()` in the same order; each is three kernels on the context
    stream (asynchronous, graph-capturable)."""

    def __init__(self, dec: "SlabDecomposition", ops):
        import torch

        self.dec, self.ops = dec, ops
        lay = dec.lay
        self.count = lay.local_planes * lay.plane
        lib = load()
        self._ptrs = []
        for _ in range(2):
            ptr = C.c_void_p()
            check(lib.ibc_device_alloc(ops.context.handle, self.count * 8, C.byref(ptr)))
            self._ptrs.append(ptr.value)
        sig = C.c_void_p()
        check(lib.ibc_slab_signals_create(ops.context.handle, C.byref(sig)))
        self._sig = sig.value
        dev = torch.device("cuda", ops.device)
        self.spread_buf = torch.as_tensor(_DeviceArray(self._ptrs[0], self.count), device=dev)
        self.field_buf = torch.as_tensor(_DeviceArray(self._ptrs[1], self.count), device=dev)
        self.field_buf.zero_()
        self._opened = []
        self._links = None

    def _link(self, which: int, down, up) -> _capi.IbcSlabLink:
        lay = self.dec.lay
        L = _capi.IbcSlabLink()
        L.nloc = lay.nloc
        L.nloc_down = down[3]
        L.plane = lay.plane
        L.has_down = int(self.dec._has_down())
        L.has_up = int(self.dec._has_up())
        L.d_local = self._ptrs[which]
        L.d_down = down[which]
        L.d_up = up[which]
        L.d_sig = self._sig
        L.d_sig_down = down[2]
        L.d_sig_up = up[2]
        return L

    def _wire(self, down, up):
        """down / up: (spread_ptr, field_ptr, sig_ptr, nloc) of the neighbours."""
        self._links = [self._link(0, down, up), self._link(1, down, up)]

    def describe(self):
        return (self._ptrs[0], self._ptrs[1], self._sig, self.dec.lay.nloc)

    def connect_local(self, peers) -> None:
        """Ranks in one process: peers[r] is rank r's PeerSlab."""
        self._wire(peers[self.dec.down].describe(), peers[self.dec.up].describe())

    def connect_ipc(self, group=None) -> None:
        """One process per rank: swap IPC handles over the process group."""
        import torch.distributed as dist

        lib, h = load(), self.ops.context.handle
        mine = []
        for ptr in (*self._ptrs, self._sig):
            hd = _capi.IbcIpcHandle()
            check(lib.ibc_ipc_get_handle(h, C.c_void_p(ptr), C.byref(hd)))
            mine.append(bytes(hd.bytes))
        allh = [None] * self.dec.lay.world
        dist.all_gather_object(allh, (mine, self.dec.lay.nloc), group=group)
        opened = {}

        def peer(r):
            if r == self.dec.lay.rank:
                return self.describe()
            if r not in opened:
                ptrs = []
                for raw in allh[r][0]:
                    hd = _capi.IbcIpcHandle()
                    C.memmove(hd.bytes, raw, 64)
                    out = C.c_void_p()
                    check(lib.ibc_ipc_open_handle(h, C.byref(hd), C.byref(out)))
                    ptrs.append(out.value)
                    self._opened.append(out.value)
                opened[r] = (*ptrs, allh[r][1])
            return opened[r]

        self._wire(peer(self.dec.down), peer(self.dec.up))

    def _exchange(self, fn, which):
        if self._links is None:
            raise RuntimeError("PeerSlab is not connected (connect_ipc / connect_local)")
        self.ops._sync_stream()
        # epoch 0: the device-side counter -- correct under CUDA graph replay
        check(fn(self.ops.context.handle, C.byref(self._links[which]), 0))

    def ghost_sum(self):
        """spread_buf: local spread output -> its owned planes ghost-summed."""
        self._exchange(load().ibc_slab_ghost_sum_device, 0)
        lay = self.dec.lay
        return self.spread_buf[2 * lay.plane:(lay.nloc + 2) * lay.plane]

    def halo_fill(self):
        """field_buf: owned planes (written by the caller) -> halos filled."""
        self._exchange(load().ibc_slab_halo_fill_device, 1)
        return self.field_buf

    @property
    def owned_field(self):
        """The owned planes of field_buf (write the rank's field here)."""
        lay = self.dec.lay
        return self.field_buf[2 * lay.plane:(lay.nloc + 2) * lay.plane]

    def timed_out(self) -> bool:
        flag = C.c_int()
        check(load().ibc_slab_link_error(self.ops.context.handle, C.byref(self._links[0]),
                                         C.byref(flag)))
        return bool(flag.value)

    def close(self) -> None:
        lib = load()
        h = getattr(self.ops, "context", None)
        if h is None or not getattr(self, "_ptrs", None):
            return
        for p in self._opened:
            lib.ibc_ipc_close_handle(h.handle, C.c_void_p(p))
        for p in (*self._ptrs, self._sig):
            lib.ibc_device_free(h.handle, C.c_void_p(p))
        self._ptrs, self._opened = [], []
