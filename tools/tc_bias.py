"""Diagnose the 3xTF32 GEMM error: signed relative error vs n (accumulation chain length)."""
import numpy as np, torch
from paper_2402_08134_b200 import symnmf as S
torch.backends.cuda.matmul.allow_tf32 = False
rng = np.random.default_rng(0)
for n in (2048, 8192, 30000):
    for kind in ("exact-tf32", "uniform"):
        if kind == "exact-tf32":
            A = (rng.integers(1, 1024, size=(n, n)) / 1024).astype(np.float32)   # <= 10 mantissa bits
            X = (rng.integers(1, 1024, size=(n, 32)) / 1024).astype(np.float32)
        else:
            A = rng.random((n, n), dtype=np.float32); X = rng.random((n, 32), dtype=np.float32)
        M = S.DeviceMatrix.from_host(A)
        Y = S.ah(M, torch.from_numpy(X).cuda(), precision="3xtf32").cpu().numpy().astype(np.float64)
        ref = A.astype(np.float64) @ X.astype(np.float64)
        Yf = (torch.from_numpy(A).cuda() @ torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
        e = (Y - ref) / ref
        ef = (Yf - ref) / ref
        print(f"n={n:6d} {kind:10s} tc: mean {e.mean():+.3e} max|.| {np.abs(e).max():.3e}   "
              f"fp32 sgemm: mean {ef.mean():+.3e} max {np.abs(ef).max():.3e}", flush=True)
        del M
