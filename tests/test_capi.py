"""The C-ABI library loads and exports exactly what include/ibcuda.h declares
(CPU; no compute calls)."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2012_06646_b200 import _capi
from paper_2012_06646_b200 import ib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "ibcuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ibc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _capi.load()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_capi.SIGNATURES), "ctypes binding out of sync with ibcuda.h"
    assert lib.ibc_version() == 1


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_capi.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_grid_validation_mirrors_staggered_grid_ctor():
    # tests/grid_test.cpp:184-196
    with pytest.raises(ib.InvalidArgument):
        ib.StaggeredGrid([0], 1.0, [0.0], [False])
    with pytest.raises(ib.InvalidArgument):
        ib.StaggeredGrid([4], 0.0, [0.0], [False])
    with pytest.raises(ib.InvalidArgument):
        ib.StaggeredGrid([4], 1.0, [1.0], [False])
    with pytest.raises(ib.InvalidArgument):
        ib.StaggeredGrid([4], 1.0, [-0.1], [False])
    with pytest.raises(ib.LengthError):
        ib.StaggeredGrid([70000, 70000], 1.0, [0.0, 0.0], [True, True])
    ib.StaggeredGrid([65000, 65000], 1.0, [0.0, 0.0], [True, True])


def test_grid_accessors():
    g = ib.StaggeredGrid([4, 6], 0.5, [0.0, 0.5], [True, False], [1.0, 2.0])
    assert g.point_count() == 24
    assert g.axis_length(1) == 3.0
    assert g.is_periodic(0) and not g.is_periodic(1)
    assert g.staggering(1) == 0.5 and g.spacing() == 0.5


def test_vector_spread_checks_run_before_any_device_work():
    # ib.spread_vector checks every component's arguments first, in the
    # reference's order (spread.hpp:321-350 -> :60-77, :314); these cases fail
    # at component 0, so no library call (and no GPU) is needed
    g = [ib.StaggeredGrid([8, 8], 0.5, a, [True, True]) for a in ([0.0, 0.5], [0.5, 0.0])]
    pts = np.array([[1.0, 1.0], [2.0, 2.0]])
    vals = [np.ones(2), np.ones(2)]
    K = ib.CosineKernel()
    with pytest.raises(ib.InvalidArgument, match="one grid per vector component"):
        ib.spread_vector(pts, vals, g[:1], K, ib.SpreadAlgorithm.serial, 0, None, 1)
    with pytest.raises(ib.InvalidArgument, match="fused spreading needs a workspace"):
        ib.spread_vector(pts, vals, g, K, ib.SpreadAlgorithm.fused, 0, None, 1)
    with pytest.raises(ib.InvalidArgument, match="buffered spreading needs a workspace"):
        ib.spread_vector(pts, vals, g, K, ib.SpreadAlgorithm.buffered, 0, None, 1)
    with pytest.raises(ib.InvalidArgument, match="sweep width must be >= 1"):
        ib.spread_vector(pts, vals, g, K, ib.SpreadAlgorithm.otf, 0, None, 1)
    with pytest.raises(ib.InvalidArgument, match="one value per point"):
        ib.spread_vector(pts, [np.ones(3), np.ones(2)], g, K, ib.SpreadAlgorithm.serial, 0, None, 1)
    with pytest.raises(ib.InvalidArgument, match="unknown spreading algorithm"):
        ib.spread_vector(pts, vals, g, K, 7, 0, None, 1)
    with pytest.raises(ib.InvalidArgument, match="expected one field per vector component"):
        ib.interpolate_vector([ib.GridField(g[0])], pts, K, 1)
