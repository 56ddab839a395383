"""B200-native Spreeze (arXiv 2312.06126) network-update hot path.

The product is ``libspz.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/spz.h``); ``spz`` is its ctypes binding.  Build with
``python -m paper_2312_06126_b200.build``.
"""

from . import spz  # noqa: F401
from .spz import Learner, Replay, SpzError  # noqa: F401
