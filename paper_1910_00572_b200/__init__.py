"""gridloc_b200 — B200-native map-corrected-odometry belief filter.

Drop-in for the hot path of the reference ``gridloc`` library
(arXiv:1910.00572): map load, belief init, the Algorithm-1 predict/correct
step, belief map / argmax, Floyd-Steinberg sample extraction and the sampled
LIDAR update. The FP64 belief tensor lives in HBM; every tensor operation is
a hand-written sm_100a kernel in ``libgridloc_b200.so`` behind the C-ABI of
``include/gridloc_b200.h``.

The library is mapped on first use (the first Context / map / kernel-set
call), not at import, so that input generators (``floorplan``) can be
imported by the reference arm of bench.py without mapping the product. That
first use fails loudly when the library is missing: there is no CPU
fallback. ``load_native()`` maps it eagerly.
"""
from . import _lib
from .gridloc import *  # noqa: E402,F401,F403
from .gridloc import tensor_hash_host, tensor_status, tensors_status  # noqa: E402,F401

__version__ = "0.2.0"


def load_native():
    """Map libgridloc_b200.so now (raises ImportError if it is absent)."""
    return _lib.load()
