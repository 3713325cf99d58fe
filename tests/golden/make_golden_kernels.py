"""Golden fixtures for the kernels beyond CosineKernel, from the REFERENCE.

The reference's operators are templates over any `Kernel` (kernel.hpp:16-21);
oracle/ref_driver.cpp instantiates them with Peskin's 4-point kernel, the
3-point kernel of Roma, Peskin & Berger (odd support: cell_index half = 0.5,
grid.hpp:121-130) and the 2-point hat, written as the reference's own tests
write their kernels (tests/grid_test.cpp:18-23).  This script freezes the
reference's outputs for them (golden_kernels.npz: 40 random cases, D in
{1,2,3}, mixed periodicity / staggering / origin, kernel ids 0..3 of
include/ibcuda.h) -- spread_fused field + ws.keys / ws.perm / ws.run_keys,
spread_serial field and interpolate output.

    python tests/golden/make_golden_kernels.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
import oracle as O  # noqa: E402


def main():
    assert O.ref_available(), "oracle/_ref/libibref.so missing: run make -C oracle"
    rng = np.random.default_rng(2012_06646 + 4)
    out = {}
    ncases = 40
    for c in range(ncases):
        kernel = c % 4
        d = 1 + (c // 4) % 3
        ext = rng.integers(3, 14, d)
        alpha = rng.choice([0.0, 0.25, 0.5, 0.7], d)
        per = rng.integers(0, 2, d)
        h = float(rng.uniform(0.3, 0.9))
        origin = rng.uniform(-1.0, 1.0, d)
        n = int(rng.integers(0, 400))
        pts = np.empty((n, d))
        for a in range(d):
            L = ext[a] * h
            pts[:, a] = origin[a] + (rng.uniform(-L, 2 * L, n) if per[a] else rng.uniform(0.0, L, n))
        vals = rng.uniform(-1.0, 1.0, n)
        g = O.make_grid(ext, h, alpha, per, origin)
        field, keys, perm, run_keys = O.ref_spread(g, pts, vals, "fused", workers=1 + c % 3,
                                                   kernel=kernel)
        serial, *_ = O.ref_spread(g, pts, vals, "serial", kernel=kernel)
        e = rng.uniform(-1.0, 1.0, O.grid_points(g))
        interp = O.ref_interpolate(g, e, pts, workers=2, kernel=kernel)
        p = f"c{c}_"
        out.update({p + "kernel": np.array([kernel]), p + "ext": ext, p + "h": np.array([h]),
                    p + "alpha": alpha, p + "per": per, p + "origin": origin, p + "pts": pts,
                    p + "vals": vals, p + "field": e, p + "spread": field, p + "keys": keys,
                    p + "perm": perm, p + "run_keys": run_keys, p + "serial": serial,
                    p + "interp": interp})
    out["ncases"] = np.array([ncases])
    np.savez_compressed(HERE / "golden_kernels.npz", **out)
    print("wrote", HERE / "golden_kernels.npz")


if __name__ == "__main__":
    main()
