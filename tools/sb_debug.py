"""Debug run of the tensor-core sampled dense product on a tiny case (SYMNMF_SB_DEBUG=1 prints)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from synth import random_factor  # noqa: E402
from paper_2402_08134_b200 import symnmf as S  # noqa: E402

n, k, s = 256, 32, 64
r = np.random.default_rng(1)
X = r.random((n, n))
A = ((X + X.T) / 2).astype(np.float32)
F = random_factor(n, k, 11) ** 2
lev = O.leverage_scores(F).astype(np.float32)
plan = S.hybrid_sample(torch.from_numpy(lev).cuda(), k, s, 1.0 / s, 3, 1, 0)
o = O.build_plan(lev, k, s, 1.0 / s, 3, 1, 0)
Gr, Yr = O.sampled_products(A, F, o["uniq_idx"], o["uniq_w"])
M = S.DeviceMatrix.from_host(A)
print("n_uniq", o["n_uniq"], "Yr[0,:3]", Yr[0, :3], "Yr[32,0]", Yr[32, 0], flush=True)
Y, _ = S.sampled_ah(M, torch.from_numpy(F).cuda(), plan)
torch.cuda.synchronize()
Yg = Y.cpu().numpy()
print("Y[0,:3]", Yg[0, :3], "Y[32,0]", Yg[32, 0], "rel", np.linalg.norm(Yg - Yr) / np.linalg.norm(Yr), flush=True)
