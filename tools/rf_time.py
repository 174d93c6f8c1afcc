import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2402_08134_b200 import symnmf as S
from synth import make_input
d = make_input("c5"); cfg = d["cfg"]
M = S.DeviceMatrix.from_host(d["A"])
for prec in ("3xtf32", "fp32"):
    for rep in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        U, lam = S.rangefinder(M, cfg.l, cfg.q, cfg.seed, precision=prec)
        torch.cuda.synchronize(); print(prec, rep, "rangefinder s", time.perf_counter() - t, flush=True)
