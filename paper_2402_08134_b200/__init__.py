"""B200-native (sm_100a) hot path of randomized SymNMF (arXiv 2402.08134).

The product is libsymnmf.so (CUDA kernels + C ABI, include/symnmf.h); the
PyTorch binding is `paper_2402_08134_b200.symnmf`.  Importing this package
does not require a GPU; calling any operation does, and fails loudly without
the built library.
"""
from ._abi import (DENSE, CSR, FP32, TF32X3, EXACT, LVS, LAI, SymNMFError, load as load_library,  # noqa: F401
                   LIB_PATH)

__all__ = ["load_library", "LIB_PATH", "SymNMFError"]
