"""lmscale: B200-native uniqueness embedding-gradient exchange (arXiv 1810.10045 Sec. 3.1).

The compute path is ``liblmscale.so`` (hand-written CUDA for sm_100a + NCCL)
behind the C ABI in ``include/lmscale.h``; ``lmscale`` is its ctypes binding.
Importing the binding raises if the library has not been built -- there is
no CPU fallback.
"""
from .lmscale import (Context, LmscaleError, SparseGrad, get_nccl_id, version,  # noqa: F401
                      FLAG_NO_COMM, FLAG_TIMING, FLAG_GRAPH, LIB_PATH)
from . import distributed  # noqa: F401
