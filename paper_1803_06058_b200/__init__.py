"""B200-native LOVE (LanczOs Variance Estimates, arXiv 1803.06058) for KISS-GP.

The method runs in liblove.so (hand-written CUDA for sm_100a behind the C ABI of
include/love.h); this package is the thin Python binding.  See DESIGN.md.
"""
from .love import LoveCache, LoveError, build_cache, launch_count, nccl_unique_id  # noqa: F401
from ._abi import LIB_PATH  # noqa: F401
