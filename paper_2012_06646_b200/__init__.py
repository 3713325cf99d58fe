"""B200-native immersed-boundary spread / interpolate (arXiv 2012.06646).

The hot path -- cell keys, onesweep key/index sort, write-once tiled spread,
interpolation gather -- is CUDA for sm_100a in ``csrc/``, built into
``_lib/libibcuda.so`` behind the C ABI of ``include/ibcuda.h``.

* ``paper_2012_06646_b200.ib``      -- the reference's operator API (host buffers)
* ``paper_2012_06646_b200.device``  -- device-resident operators on torch tensors
* ``paper_2012_06646_b200.slab``    -- z-slab decomposition across GPUs
"""
from ._capi import LIB_PATH, load  # noqa: F401

__version__ = "0.1.0"
