"""Quick check of both sampled dense products (tensor-core and SIMT) against the oracle, before the
full parity tests."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from synth import random_factor  # noqa: E402
from paper_2402_08134_b200 import symnmf as S  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


for n, k, s in [(1000, 8, 200), (3000, 32, 1500), (2052, 64, 700)]:
    r = np.random.default_rng(n)
    X = r.random((n, n))
    A = ((X + X.T) / 2).astype(np.float32)
    F = random_factor(n, k, 11) ** 2
    lev = O.leverage_scores(F).astype(np.float32)
    plan = S.hybrid_sample(torch.from_numpy(lev).cuda(), k, s, 1.0 / s, 3, 1, 0)
    o = O.build_plan(lev, k, s, 1.0 / s, 3, 1, 0)
    Gr, Yr = O.sampled_products(A, F, o["uniq_idx"], o["uniq_w"])
    M = S.DeviceMatrix.from_host(A)
    for env in ({"SYMNMF_SAMPLED_DENSE": "tc"}, {"SYMNMF_SAMPLED_DENSE": "simt"}):
        os.environ.update(env)
        try:
            Y, _ = S.sampled_ah(M, torch.from_numpy(F).cuda(), plan)
            torch.cuda.synchronize()
            print(n, k, s, env, "rel", rel(Y.cpu().numpy(), Yr), flush=True)
        except Exception as e:  # noqa: BLE001
            print(n, k, s, env, "ERR", e, flush=True)
