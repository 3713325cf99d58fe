"""Regenerate the golden fixtures from the REFERENCE itself.

Runs the unmodified reference headers, compiled in place by oracle/Makefile
into oracle/_ref/libibref.so (requires /root/reference at build time).  The
outputs frozen here pin both the C restatement (tests/test_oracle.py, CPU)
and the CUDA path (tests/test_gpu_parity.py):

* golden_small.npz -- 48 random small cases, D in {1,2,3}, mixed periodicity
  and staggering, points straddling periodic boundaries (the shape of
  tests/coupling_test.cpp:240-283): inputs + spread_fused field, ws.keys,
  ws.perm, ws.run_keys, spread_serial field, interpolate output.  Plus the
  spread walkthrough of tests/coupling_test.cpp:205-217.
* golden_c1.json   -- BASELINE config 1 (2^16 scatter_points, 64^3, alpha =
  (1/2, 1/2, 0)): SHA-256 of ws.keys / ws.perm, q, and value checksums.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
import oracle as O  # noqa: E402


def random_case(rng, d):
    ext = rng.integers(4, 13, d)
    alpha = rng.uniform(0.0, 0.999, d)
    per = rng.integers(0, 2, d)
    h = 0.5
    n = int(rng.integers(0, 301))
    pts = np.empty((n, d))
    for a in range(d):
        L = ext[a] * h
        pts[:, a] = rng.uniform(-L, 2 * L, n) if per[a] else rng.uniform(0.0, L, n)
    vals = rng.uniform(-1.0, 1.0, n)
    return ext, h, alpha, per, pts, vals


def main():
    assert O.ref_available(), "oracle/_ref/libibref.so missing: run make -C oracle"
    rng = np.random.default_rng(20126646)
    out = {}
    cases = []
    for c in range(48):
        d = 1 + c % 3
        ext, h, alpha, per, pts, vals = random_case(rng, d)
        g = O.make_grid(ext, h, alpha, per)
        field, keys, perm, run_keys = O.ref_spread(g, pts, vals, "fused", workers=1 + c % 4)
        serial, *_ = O.ref_spread(g, pts, vals, "serial")
        e = rng.uniform(-1.0, 1.0, O.grid_points(g))
        interp = O.ref_interpolate(g, e, pts, workers=2)
        p = f"c{c}_"
        out.update({p + "ext": ext, p + "h": np.array([h]), p + "alpha": alpha, p + "per": per,
                    p + "pts": pts, p + "vals": vals, p + "field": e, p + "spread": field,
                    p + "keys": keys, p + "perm": perm, p + "run_keys": run_keys,
                    p + "serial": serial, p + "interp": interp})
        cases.append(c)
    # Spread walkthrough (tests/coupling_test.cpp:205-217).
    g = O.make_grid([4, 4], 1.0, [0.0, 0.0], [0, 0])
    pts = np.array([[0.6, 0.6], [2.3, 1.1], [1.8, 1.3], [2.2, 0.4], [1.1, 1.1]])
    vals = np.array([1.0, 2.0, 4.0, 8.0, 16.0])
    field, keys, perm, run_keys = O.ref_spread(g, pts, vals, "fused", workers=2)
    out.update({"walk_pts": pts, "walk_vals": vals, "walk_spread": field, "walk_keys": keys,
                "walk_perm": perm, "walk_run_keys": run_keys})
    out["ncases"] = np.array([len(cases)])
    np.savez_compressed(HERE / "golden_small.npz", **out)

    # BASELINE config 1.
    n, N, edge = 1 << 16, 64, 16e-4
    h = edge / N
    g = O.make_grid([N] * 3, h, [0.5, 0.5, 0.0], [1, 1, 1])
    pts = O.scatter_points(n, edge, 1)
    ref_pts = np.zeros(n * 3)
    O.ref().ref_scatter_points(n, edge, 1, ref_pts)
    assert np.array_equal(pts.reshape(-1), ref_pts)
    vals = 2.0 * O.scatter_points(n, 1.0, 2)[:, 0] - 1.0
    field, keys, perm, run_keys = O.ref_spread(g, pts, vals, "fused", workers=8)
    e = 2.0 * O.scatter_points(N ** 3 // 3 + 1, 1.0, 4).reshape(-1)[: N ** 3] - 1.0
    interp = O.ref_interpolate(g, e, pts, workers=8)
    c1 = {
        "n": n, "N": N, "edge_cm": edge, "alpha": [0.5, 0.5, 0.0],
        "keys_sha256": hashlib.sha256(keys.tobytes()).hexdigest(),
        "perm_sha256": hashlib.sha256(perm.tobytes()).hexdigest(),
        "run_keys_sha256": hashlib.sha256(run_keys.tobytes()).hexdigest(),
        "run_count": int(run_keys.size),
        "spread_sum": float(field.sum()), "spread_abs_max": float(np.abs(field).max()),
        "spread_l2": float(np.sqrt((field ** 2).sum())),
        "interp_sum": float(interp.sum()), "interp_abs_max": float(np.abs(interp).max()),
        "generator": "points = scatter_points(n, edge, 1) (bench/setup.hpp:46-53); "
                     "values = 2*scatter_points(n, 1, 2)[:,0]-1; "
                     "field = 2*scatter_points(N^3/3+1, 1, 4).flat[:N^3]-1",
    }
    (HERE / "golden_c1.json").write_text(json.dumps(c1, indent=1) + "\n")
    print("wrote", HERE / "golden_small.npz", HERE / "golden_c1.json", "q(c1) =", c1["run_count"])


if __name__ == "__main__":
    main()
