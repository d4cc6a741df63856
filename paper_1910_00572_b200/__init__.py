"""gridloc_b200 — B200-native map-corrected-odometry belief filter.

Drop-in for the hot path of the reference ``gridloc`` library
(arXiv:1910.00572): map load, belief init, the Algorithm-1 predict/correct
step, belief map / argmax, Floyd-Steinberg sample extraction and the sampled
LIDAR update. The FP64 belief tensor lives in HBM; every tensor operation is
a hand-written sm_100a kernel in ``libgridloc_b200.so`` behind the C-ABI of
``include/gridloc_b200.h``. Importing this package fails loudly when that
library is missing: there is no CPU fallback.
"""
from . import _lib

_lib.load()  # fail loudly at import when the native library is absent

from .gridloc import *  # noqa: E402,F401,F403
from .gridloc import tensor_hash_host, tensor_status  # noqa: E402,F401

__version__ = "0.1.0"
