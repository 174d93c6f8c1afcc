"""B200-native (sm_100a) hot path of randomized SymNMF (arXiv 2402.08134).

The product is libsymnmf.so (CUDA kernels + C ABI, include/symnmf.h); this
package is its thin PyTorch binding.  Importing it does not require a GPU;
calling any operation does, and fails loudly without the built library.
"""
from ._abi import (DENSE, CSR, FP32, TF32X3, EXACT, LVS, LAI, SymNMFError, load as load_library,  # noqa: F401
                   LIB_PATH)

__all__ = ["load_library", "LIB_PATH", "SymNMFError"]


def __getattr__(name):
    # the torch-dependent binding is imported lazily
    from . import symnmf as _s
    if hasattr(_s, name):
        return getattr(_s, name)
    raise AttributeError(name)
