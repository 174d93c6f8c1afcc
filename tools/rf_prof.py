"""Two warm calls of the range finder on c5 (for an ncu launch list of its kernels)."""
import sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2402_08134_b200 import symnmf as S  # noqa: E402
from synth import make_input  # noqa: E402
d = make_input("c5"); cfg = d["cfg"]
M = S.DeviceMatrix.from_host(d["A"])
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    U, lam = S.rangefinder(M, cfg.l, cfg.q, cfg.seed, precision="3xtf32")
    e1.record(); torch.cuda.synchronize()
    print("rangefinder ms", e0.elapsed_time(e1), flush=True)
