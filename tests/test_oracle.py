"""Pin the parity oracle (CPU, no GPU needed).

The C restatement (oracle/ib_oracle.c) must reproduce (1) the reference's own
known-answer tests and (2) the golden vectors produced by the reference
headers themselves (tests/golden/make_golden.py).  Only then is it trusted as
the checker of the CUDA path.
"""
import ctypes as C
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"


def ints(*v):
    return (C.c_int * len(v))(*v)


def test_cell_index_kats():
    # tests/grid_test.cpp:30-34 (even support associates the point at or above x)
    g = O.make_grid([8], 1.0, [0.0], [0])
    out = (C.c_int * 1)()
    O.lib().or_cell_index(C.byref(g), (C.c_double * 1)(2.6), 4, out)
    assert out[0] == 3
    O.lib().or_cell_index(C.byref(g), (C.c_double * 1)(2.0), 4, out)
    assert out[0] == 2
    # grid_test.cpp:36-44 (odd support: nearest grid point)
    g2 = O.make_grid([8, 8], 0.5, [0.0, 0.5], [0, 0])
    out2 = (C.c_int * 2)()
    O.lib().or_cell_index(C.byref(g2), (C.c_double * 2)(1.3, 0.9), 3, out2)
    assert list(out2) == [3, 1]


def test_grid_index_and_keys_kats():
    per = O.make_grid([4, 4], 1.0, [0.0, 0.0], [1, 1])
    closed = O.make_grid([4, 4], 1.0, [0.0, 0.0], [0, 0])
    L = O.lib()
    assert L.or_grid_index(C.byref(per), ints(-1, 2)) == 11          # grid_test.cpp:82
    assert L.or_grid_index(C.byref(closed), ints(-1, 2)) == 0xFFFFFFFF  # :83
    assert L.or_cell_key(C.byref(per), ints(0, 0)) == 7               # :101
    assert L.or_cell_key(C.byref(closed), ints(0, 0)) == 7            # :102
    assert L.or_cell_key(C.byref(per), ints(-1, 0)) == L.or_cell_key(C.byref(per), ints(3, 0))
    assert L.or_cell_key(C.byref(per), ints(4, 2)) == L.or_cell_key(C.byref(per), ints(0, 2))
    back = (C.c_int * 2)()
    L.or_cell_key_inverse(C.byref(per), L.or_cell_key(C.byref(per), ints(-1, 2)), back)
    assert list(back) == [3, 2]                                        # :137-138


def test_cell_key_round_trip_and_colex_monotone():
    # grid_test.cpp:105-124
    g = O.make_grid([5, 5, 5], 1.0, [0.0] * 3, [0, 0, 0])
    L = O.lib()
    prev = -1
    back = (C.c_int * 3)()
    for iz in range(-1, 6):
        for iy in range(-1, 6):
            for ix in range(-1, 6):
                k = L.or_cell_key(C.byref(g), ints(ix, iy, iz))
                L.or_cell_key_inverse(C.byref(g), k, back)
                assert list(back) == [ix, iy, iz]
                assert k > prev
                prev = k


def test_kernel_and_shift_kats():
    L = O.lib()
    assert L.or_cosine_phi(0.0) == 0.5                                 # kernel_test.cpp:16-22
    assert L.or_cosine_phi(1.0) == pytest.approx(0.25, abs=1e-16)
    assert L.or_cosine_phi(2.0) == 0.0 and L.or_cosine_phi(-2.0) == 0.0
    s = (C.c_int * 3)()
    L.or_shift(3, 1, 4, s)
    assert list(s) == [-2, -2, -2]                                     # kernel_test.cpp:79-84
    L.or_shift(3, 64, 4, s)
    assert list(s) == [1, 1, 1]
    s2 = (C.c_int * 2)()
    L.or_shift(2, 5, 3, s2)
    assert list(s2) == [0, 0]
    rng = np.random.default_rng(3)
    for x in rng.uniform(0, 1, 200):                                   # partition of unity
        assert sum(L.or_cosine_phi(x - j) for j in range(-3, 4)) == pytest.approx(1.0, abs=1e-14)


def test_sort_walkthrough_and_reduce():
    # Fig. 3 walkthrough (inc/bench/verify.hpp:234-256; primitives_test.cpp:48-54)
    keys = np.array([1, 6, 5, 3, 5], np.uint32)
    perm = np.array([1, 2, 3, 4, 5], np.uint32)
    O.lib().or_key_value_sort(keys, perm, 5)
    assert keys.tolist() == [1, 3, 5, 5, 6]
    assert perm.tolist() == [1, 4, 3, 5, 2]
    vals = np.array([2.0, 4.0, 8.0, 16.0, 32.0])[perm - 1]
    ok = np.zeros(5, np.uint32)
    os_ = np.zeros(5)
    q = O.lib().or_segmented_reduce(keys, vals, 5, ok, os_)
    assert q == 4 and ok[:4].tolist() == [1, 3, 5, 6] and os_[:4].tolist() == [2.0, 16.0, 40.0, 4.0]


def test_sort_matches_stable_sort_and_reference():
    # primitives_test.cpp:71-94 shape: random sizes, narrow key ranges force duplicates
    rng = np.random.default_rng(101)
    for trial in range(300):
        n = int(rng.integers(0, 1001))
        hi = 40 if trial % 2 else 0xFFFFFFFE
        keys = rng.integers(0, hi + 1, n, dtype=np.uint64).astype(np.uint32)
        pay = np.arange(n, dtype=np.uint32)
        order = np.argsort(keys, kind="stable")
        k1, p1 = keys.copy(), pay.copy()
        O.lib().or_key_value_sort(k1, p1, n)
        assert np.array_equal(k1, keys[order]) and np.array_equal(p1, pay[order])
        if O.ref_available():
            k2, p2 = keys.copy(), pay.copy()
            O.ref().ref_key_value_sort(k2, p2, n, 1 + trial % 8)
            assert np.array_equal(k1, k2) and np.array_equal(p1, p2)


def _golden():
    return np.load(GOLD / "golden_small.npz")


def test_oracle_matches_reference_golden_vectors():
    z = _golden()
    for c in range(int(z["ncases"][0])):
        p = f"c{c}_"
        g = O.make_grid(z[p + "ext"], float(z[p + "h"][0]), z[p + "alpha"], z[p + "per"])
        pts, vals = z[p + "pts"], z[p + "vals"]
        field, keys, perm, run_keys = O.spread_fused(g, pts, vals)
        assert np.array_equal(keys, z[p + "keys"]), c
        assert np.array_equal(perm, z[p + "perm"]), c
        assert np.array_equal(run_keys, z[p + "run_keys"]), c
        assert O.max_rel_deviation(field, z[p + "spread"]) <= 1e-12, c
        assert np.array_equal(O.spread_serial(g, pts, vals), z[p + "serial"]), c
        assert np.array_equal(O.interpolate(g, z[p + "field"], pts), z[p + "interp"]), c


def test_oracle_spread_walkthrough():
    # tests/coupling_test.cpp:205-217
    z = _golden()
    g = O.make_grid([4, 4], 1.0, [0.0, 0.0], [0, 0])
    field, keys, perm, run_keys = O.spread_fused(g, z["walk_pts"], z["walk_vals"])
    assert perm.tolist() == [0, 3, 2, 4, 1]
    assert run_keys.size == 4
    assert np.array_equal(keys, z["walk_keys"])
    assert O.max_rel_deviation(field, z["walk_spread"]) <= 1e-12


def test_oracle_config1_hashes():
    c1 = json.loads((GOLD / "golden_c1.json").read_text())
    n, N, edge = c1["n"], c1["N"], c1["edge_cm"]
    g = O.make_grid([N] * 3, edge / N, c1["alpha"], [1, 1, 1])
    pts = O.scatter_points(n, edge, 1)
    keys, perm, run_keys = O.prepare_keys(g, pts)
    assert hashlib.sha256(keys.tobytes()).hexdigest() == c1["keys_sha256"]
    assert hashlib.sha256(perm.tobytes()).hexdigest() == c1["perm_sha256"]
    assert run_keys.size == c1["run_count"] == 58038


def test_oracle_invariants():
    # adjointness + conservation (tests/coupling_test.cpp:326-375)
    rng = np.random.default_rng(73)
    g = O.make_grid([8, 8, 8], 0.5, [0.0, 0.5, 0.5], [1, 0, 1])
    hd = 0.5 ** 3
    for _ in range(5):
        pts = np.stack([rng.uniform(-4, 8, 120), rng.uniform(0, 4, 120), rng.uniform(-4, 8, 120)], 1)
        w = rng.uniform(-1, 1, 120)
        e = rng.uniform(-1, 1, 512)
        grid_side = hd * float(O.spread_serial(g, pts, w) @ e)
        interp = O.interpolate(g, e, pts)
        point_side = float(w @ interp)
        assert abs(grid_side - point_side) <= 1e-12 * float(np.abs(w * interp).sum())


# ------------------------------------------------------------------ other kernels
def test_kernel_kats():
    # Peskin 4-point: phi(0) = 1/2, phi(1) = 1/4, phi(2) = 0 (as kernel_test.cpp:16-22
    # pins the cosine kernel); Roma 3-point: phi(0) = 2/3, phi(1) = 1/6, phi(3/2) = 0;
    # hat: phi(0) = 1, phi(1/2) = 1/2, phi(1) = 0.
    for k, r, want in [(0, 0.0, 0.5), (0, 1.0, 0.25), (0, 2.0, 0.0), (1, 0.0, 0.5), (1, 1.0, 0.25),
                       (1, -1.0, 0.25), (1, 2.0, 0.0), (2, 0.0, 2 / 3), (2, 1.0, 1 / 6),
                       (2, 1.5, 0.0), (3, 0.0, 1.0), (3, 0.5, 0.5), (3, 1.0, 0.0)]:
        assert O.kernel_phi(k, r) == pytest.approx(want, abs=1e-15), (k, r)
    assert [O.lib().or_kernel_support(k) for k in range(5)] == [4, 4, 3, 2, 0]
    # zeroth moment and the even/odd split every 4-point kernel satisfies
    rng = np.random.default_rng(3)
    for k in range(4):
        s = O.lib().or_kernel_support(k)
        for u in rng.uniform(0.0, 1.0, 50):
            w = [O.kernel_phi(k, j + u) for j in range(-s, s + 1)]
            assert sum(w) == pytest.approx(1.0, abs=1e-14)
        if s == 4:
            for u in rng.uniform(0.0, 1.0, 50):
                w = [O.kernel_phi(k, -2 + u + j) for j in range(4)]
                assert w[0] + w[2] == pytest.approx(0.5, abs=1e-15)
                assert w[1] + w[3] == pytest.approx(0.5, abs=1e-15)


def test_oracle_matches_reference_golden_for_every_kernel():
    z = np.load(GOLD / "golden_kernels.npz")
    for c in range(int(z["ncases"][0])):
        p = f"c{c}_"
        k = int(z[p + "kernel"][0])
        g = O.make_grid(list(z[p + "ext"]), float(z[p + "h"][0]), list(z[p + "alpha"]),
                        list(z[p + "per"]), list(z[p + "origin"]))
        pts, vals = z[p + "pts"], z[p + "vals"]
        field, keys, perm, run_keys = O.spread_fused(g, pts, vals, kernel=k)
        assert np.array_equal(keys, z[p + "keys"]), c
        assert np.array_equal(perm, z[p + "perm"]), c
        assert np.array_equal(run_keys, z[p + "run_keys"]), c
        assert O.max_rel_deviation(field, z[p + "spread"]) <= 1e-12, c
        assert O.max_rel_deviation(O.spread_serial(g, pts, vals, kernel=k), z[p + "serial"]) <= 1e-12, c
        assert O.max_rel_deviation(O.interpolate(g, z[p + "field"], pts, kernel=k), z[p + "interp"]) <= 1e-12, c
