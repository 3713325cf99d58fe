"""Synthetic IB workloads (BASELINE.json configs).

Deterministic generators, numpy-vectorized, no oracle dependency:

* ``scatter_points(n, edge, seed)`` -- bit-identical to the reference's
  ib::bench::scatter_points (bench/setup.hpp:46-53): one std::mt19937_64
  stream, x, y, z per point as (rng() >> 11) * 2^-53 * edge.
* ``uniform_pm1(count, seed)`` -- 2u - 1 from the same generator (forces,
  fields).
* ``clustered_points`` / ``rbc_points`` -- config 5 and config 4 generators.
"""
from __future__ import annotations

import math

import numpy as np

_UM = np.uint64(0xFFFFFFFF80000000)
_LM = np.uint64(0x7FFFFFFF)
_MAG = np.uint64(0xB5026F5AA96619E9)


class MT19937_64:
    """std::mt19937_64 ([rand.predef]), generating 312 words per numpy twist."""

    def __init__(self, seed: int):
        mt = np.zeros(312, dtype=np.uint64)
        mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        with np.errstate(over="ignore"):
            for i in range(1, 312):
                prev = mt[i - 1]
                mt[i] = np.uint64(6364136223846793005) * (prev ^ (prev >> np.uint64(62))) + np.uint64(i)
        self.mt = mt
        self.buf = np.zeros(0, dtype=np.uint64)

    def _twist(self) -> np.ndarray:
        mt = self.mt
        one = np.uint64(1)
        x = (mt[0:156] & _UM) | (mt[1:157] & _LM)
        mt[0:156] = mt[156:312] ^ (x >> one) ^ np.where((x & one) != 0, _MAG, np.uint64(0))
        x = (mt[156:311] & _UM) | (mt[157:312] & _LM)
        mt[156:311] = mt[0:155] ^ (x >> one) ^ np.where((x & one) != 0, _MAG, np.uint64(0))
        x = (mt[311] & _UM) | (mt[0] & _LM)
        mt[311] = mt[155] ^ (x >> one) ^ (_MAG if (x & one) else np.uint64(0))
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        return y

    def next_u64(self, count: int) -> np.ndarray:
        blocks = [self.buf]
        have = self.buf.size
        while have < count:
            b = self._twist()
            blocks.append(b)
            have += b.size
        allv = np.concatenate(blocks)
        out, self.buf = allv[:count], allv[count:]
        return out

    def next_unit(self, count: int) -> np.ndarray:
        """(rng() >> 11) * 2^-53 in [0, 1)."""
        return (self.next_u64(count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def scatter_points(n: int, edge: float, seed: int) -> np.ndarray:
    """ib::bench::scatter_points: (n, 3) uniform in [0, edge)^3."""
    return (MT19937_64(seed).next_unit(3 * n) * edge).reshape(n, 3)


def uniform_pm1(count: int, seed: int) -> np.ndarray:
    """2u - 1 in [-1, 1) (forces / field values; PCG64, fast for 10^8 draws)."""
    return np.random.Generator(np.random.PCG64(seed)).uniform(-1.0, 1.0, count)


def perturb(points: np.ndarray, amplitude: float, seed: int) -> np.ndarray:
    """X* = X + U[-amplitude, amplitude]^3 (the predicted positions of step (b))."""
    return points + uniform_pm1(points.size, seed).reshape(points.shape) * amplitude


def clustered_points(n: int, edge: float, clusters: int, sigma: float, seed: int) -> np.ndarray:
    """Config 5: n points in `clusters` Gaussian blobs (std sigma), periodic wrap."""
    rng = np.random.Generator(np.random.PCG64(seed))
    centers = rng.uniform(0.0, edge, (clusters, 3))
    which = rng.integers(0, clusters, n)
    pts = centers[which] + rng.normal(0.0, sigma, (n, 3))
    return np.mod(pts, edge)


def rbc_points(edge: float, h: float, seed: int, hematocrit_target: float = 0.4) -> np.ndarray:
    """Config 4: RBC-shaped closed surfaces (Eq. 19 of the paper).

    Biconcave disc of radius R0 = 3.91 um, z(r) = +-0.5 R0 sqrt(1 - r^2)
    (0.105 + r^2 - 0.56 r^4), sampled by a Fibonacci sphere mapped through the
    profile at ~0.8 h spacing; cells stacked in columns with small seeded
    tilts until the target volume fraction is reached.  Units: cm.
    """
    R0 = 3.91e-4
    rng = np.random.Generator(np.random.PCG64(seed))
    area = 134.2e-8  # cm^2
    per_cell = max(64, int(area / (0.8 * h) ** 2))
    i = np.arange(per_cell) + 0.5
    phi = np.arccos(1.0 - 2.0 * i / per_cell)
    theta = math.pi * (1.0 + 5.0 ** 0.5) * i
    r = np.sin(phi)
    zs = np.sign(np.cos(phi)) * 0.5 * R0 * np.sqrt(np.clip(1.0 - r * r, 0.0, 1.0)) * (
        0.105 + r * r - 0.56 * r ** 4)
    cell = np.stack([R0 * r * np.cos(theta), R0 * r * np.sin(theta), zs], axis=1)
    vol_cell = 94.4e-12  # cm^3
    n_cells = max(1, int(hematocrit_target * edge ** 3 / vol_cell))
    cols = int(math.ceil(math.sqrt(n_cells / max(1, int(edge / 2.6e-4)))))
    per_col = int(math.ceil(n_cells / (cols * cols)))
    out = []
    k = 0
    for cx in range(cols):
        for cy in range(cols):
            for cz in range(per_col):
                if k >= n_cells:
                    break
                a, b = rng.normal(0.0, 0.1, 2)
                ca, sa, cb, sb = math.cos(a), math.sin(a), math.cos(b), math.sin(b)
                rot = np.array([[cb, 0, sb], [sa * sb, ca, -sa * cb], [-ca * sb, sa, ca * cb]])
                center = np.array([(cx + 0.5) * edge / cols, (cy + 0.5) * edge / cols,
                                   (cz + 0.5) * edge / per_col])
                out.append(cell @ rot.T + center)
                k += 1
    return np.mod(np.concatenate(out), edge)


def config2(seed_offset: int = 0):
    """BASELINE config 2 at one GPU: 2^20 points, 256^3, edge 16 um."""
    n, N, edge = 1 << 20, 256, 16e-4
    h = edge / N
    xn = scatter_points(n, edge, 1 + seed_offset)
    xs = perturb(xn, 0.1 * h, 3 + seed_offset)
    g = uniform_pm1(n, 2 + seed_offset)
    e = uniform_pm1(N ** 3, 4 + seed_offset)
    return dict(n=n, N=N, edge=edge, h=h, x_n=xn, x_star=xs, values=g, field=e)


def survey_config(name: str, seed_offset: int = 0):
    """The other SURVEY 8(d) workloads in config2()'s format: c1 (2^16 points,
    64^3), w128 / w256 (one point per cell), rbc (RBC surfaces, 256^3),
    clustered (2^22 points in 64 Gaussian clusters, 512^3)."""
    edge = 16e-4
    if name == "c2":
        return config2(seed_offset)
    if name == "c1":
        N, xn = 64, scatter_points(1 << 16, edge, 1 + seed_offset)
    elif name in ("w128", "w256"):
        N = int(name[1:])
        xn = scatter_points(N ** 3, edge, 1 + seed_offset)
    elif name == "rbc":
        N = 256
        xn = rbc_points(edge, edge / N, 7 + seed_offset)
    elif name == "clustered":
        N = 512
        xn = clustered_points(1 << 22, edge, 64, 8 * edge / N, 5 + seed_offset)
    else:
        raise ValueError(f"unknown workload {name!r}")
    n, h = len(xn), edge / N
    xs = perturb(xn, 0.1 * h, 3 + seed_offset)
    return dict(n=n, N=N, edge=edge, h=h, x_n=xn, x_star=xs, values=uniform_pm1(n, 2 + seed_offset),
                field=uniform_pm1(N ** 3, 4 + seed_offset))


def slab_config(rank: int, world: int, n: int = 1 << 20):
    """Weak-scaling multi-GPU workload: a global 256 x 256 x 256*world periodic
    grid split in z-slabs of 256 planes; rank r holds n points homed in its
    slab (uniform in x, y and in its planes, kept 0.15 h inside the slab so
    X* = X^n + U[-0.1h, 0.1h] stays homed).  n = 2^20: BASELINE config 2 per
    GPU; n = 256^3: config 3's constant-load level, 1 point per cell
    (SURVEY 8(d) W, 16.8 M cells and points per GPU)."""
    N, edge = 256, 16e-4
    h = edge / N
    z0, z1 = N * rank, N * (rank + 1)
    u = MT19937_64(1 + 1000 * rank).next_unit(3 * n).reshape(n, 3)
    xn = np.empty((n, 3))
    xn[:, 0] = u[:, 0] * edge
    xn[:, 1] = u[:, 1] * edge
    # home plane of z (alpha_z = 0) is ceil(z / h): planes [z0, z1) <-> z in ((z0-1)h, (z1-1)h]
    lo, hi = (z0 - 1 + 0.15) * h, (z1 - 1 - 0.15) * h
    xn[:, 2] = lo + u[:, 2] * (hi - lo)
    xs = perturb(xn, 0.1 * h, 3 + 1000 * rank)
    g = uniform_pm1(n, 2 + 1000 * rank)
    e = uniform_pm1(N * N * N, 4 + 1000 * rank)  # this rank's owned planes
    return dict(n=n, N=N, nz_global=N * world, edge=edge, h=h, x_n=xn, x_star=xs, values=g,
                field=e, z0=z0, z1=z1)
