"""B200-native MTNUFFT hot path (arXiv 2407.01943) behind the reference's interface.

The compute lives in ``lib/libnus_b200.so`` (CUDA, sm_100a) behind the C-ABI
``include/nus_c.h``; :mod:`.api` mirrors the reference's public interface on
top of it.  There is no CPU fallback.
"""
from . import _capi
from .api import *  # noqa: F401,F403

__version__ = "0.1.0"
