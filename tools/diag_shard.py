import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_2402_08134_b200 import symnmf as S, shard as SH
from oracle import symnmf as O
from synth.configs import make_input, init_factor, mean_entry
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for cfg, n, k in [("c4", 200_000, 32), ("c4", 40_000, 32), ("c2", 100_000, 16)]:
    d = make_input(cfg, n_override=n); A = d["A"]
    H0 = init_factor(n, k, mean_entry(A), np.random.default_rng(5))
    Wr, Hr, _ = O.iterate(A, H0, H0, d["alpha"], 1, "exact")
    M = S.DeviceMatrix.from_host(A)
    for env in ["stream", "fused"]:
        import os; os.environ["SYMNMF_SWEEP"] = env
        W = torch.from_numpy(H0.copy()).cuda(); H = torch.from_numpy(H0.copy()).cuda()
        sv = S.Solver(M, W, H, d["alpha"], mode="exact", max_iters=1); sv.run(1); sv.close()
        print(cfg, n, "unsharded", env, rel(W.cpu().numpy(), Wr), rel(H.cpu().numpy(), Hr), flush=True)
    for P in [1, 2, 4]:
        sv = SH.ShardedSolver(A, H0, d["alpha"], SH.LocalComm(P), mode="exact"); sv.run(1)
        W, H = sv.factors()
        print(cfg, n, "P", P, rel(W.cpu().numpy(), Wr), rel(H.cpu().numpy(), Hr), flush=True)
