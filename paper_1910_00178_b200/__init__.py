"""B200-native u8 x i8 -> i32 GEMM (the computation NGEMM, arXiv 1910.00178, accelerates).

The product is libngemm_cuda.so (hand-written sm_100a CUDA behind the C-ABI in
include/ngemm_cuda.h).  This package is its Python front end, mirroring the reference's
C++ API (see api.py).
"""
from .api import *  # noqa: F401,F403
from .api import __all__  # noqa: F401
from ._lib import launch_count  # noqa: F401
