"""Debug: where does a free-running GPU LvS trajectory depart from the oracle's?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
from paper_2402_08134_b200 import symnmf as S
from synth import make_input

d = make_input(sys.argv[1] if len(sys.argv) > 1 else "c2")
A, H0, alpha, cfg = d["A"], d["H0"], d["alpha"], d["cfg"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
M = S.DeviceMatrix.from_host(A)
cu = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()

W1, H1 = cu(H0), cu(H0)
sv = S.Solver(M, W1, H1, alpha, mode="lvs", s=cfg.s, tau=cfg.tau, seed=0, max_iters=iters)
sv.run(iters)
st = sv.stats()["halves"]
print("solver residual", O.residual(A, H1.cpu().numpy()))

W2, H2 = cu(H0), cu(H0)
plans = {}
for it in range(iters):
    for side in (0, 1):
        F, X = (H2, W2) if side == 0 else (W2, H2)
        lev = S.leverage_scores(F)
        plan = S.hybrid_sample(lev, cfg.k, cfg.s, cfg.tau, 0, it, side)
        ph = plan.to_host()
        plans[(it, side)] = ph
        Y, Gs = S.sampled_ah(M, F, plan)
        S.hals_sweep(Gs, Y, F, X, alpha)
    print(it, "composition residual", O.residual(A, H2.cpu().numpy()), "solver stats", st[2 * it], st[2 * it + 1],
          "comp", plans[(it, 0)]["s_D"], plans[(it, 0)]["n_uniq"])
_, Hr, tr = O.iterate(A, H0, H0, alpha, iters, "lvs", s=cfg.s, tau=cfg.tau, seed=0, plans=plans)
print("oracle replaying GPU plans", O.residual(A, Hr))
_, Hr2, tr2 = O.iterate(A, H0, H0, alpha, iters, "lvs", s=cfg.s, tau=cfg.tau, seed=0)
print("oracle own plans", O.residual(A, Hr2), [t["s_D"] for t in tr2])
print("gpu s_D", [h["s_D"] for h in st])
