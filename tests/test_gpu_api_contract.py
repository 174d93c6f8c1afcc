"""GPU tests of two promises the C ABI makes (include/symnmf.h, "Asynchrony" and "Ownership"):

* the enqueue-only entry points are CUDA-graph capturable: one LvS half and one EXACT half,
  composed from the ABI calls, captured into a graph and replayed, give what the same calls
  give eagerly;
* the library keeps no global mutable state: two solvers advanced alternately on two streams
  give what each gives alone.
Comparisons are bitwise where the kernels are order-deterministic and at 1e-6 relative where
fp32 / fp64 atomics fix only the set of summands, not their order.
"""
import numpy as np
import pytest

from synth import make_input

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2402_08134_b200 import symnmf as S  # noqa: E402


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def rel(a, b):
    a = a.double().cpu().numpy() if torch.is_tensor(a) else np.asarray(a, np.float64)
    b = b.double().cpu().numpy() if torch.is_tensor(b) else np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _halves(M, F, X, alpha, k, s):
    """One LvS half and one EXACT half from the ABI calls (no host sync anywhere)."""
    lev = S.leverage_scores(F, check=False)
    plan = S.hybrid_sample(lev, k, s, 1.0 / s, 5, 3, 1, check=False)
    Ys, Gs = S.sampled_ah(M, F, plan)
    Xl = S.hals_sweep(Gs, Ys, F, X.clone(), alpha)
    Y = S.ah(M, F)
    G = S.gram(F)
    Xe = S.hals_sweep(G, Y, F, X.clone(), alpha)
    return lev, plan, Ys, Gs, Xl, Y, G, Xe


@pytest.mark.parametrize("cfgname,n", [("c2", 20_000), ("c1", 1_000)])
def test_abi_half_iterations_capture_into_a_cuda_graph(cfgname, n):
    d = make_input(cfgname, n_override=n)
    A, H0, alpha, cfg = d["A"], d["H0"], d["alpha"], d["cfg"]
    k, s = cfg.k, min(cfg.s, 400)
    M = S.DeviceMatrix.from_host(A)
    F, X = cu(H0), cu(H0 * 0.5)
    eager = _halves(M, F, X, alpha, k, s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        _halves(M, F, X, alpha, k, s)          # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(side)
    with torch.cuda.graph(g):
        cap = _halves(M, F, X, alpha, k, s)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    lev_e, plan_e, Ys_e, Gs_e, Xl_e, Y_e, G_e, Xe_e = eager
    lev_c, plan_c, Ys_c, Gs_c, Xl_c, Y_c, G_c, Xe_c = cap
    assert torch.equal(lev_c, lev_e)
    pe, pc = plan_e.to_host(), plan_c.to_host()
    assert np.array_equal(pc["uniq_idx"], pe["uniq_idx"]) and np.array_equal(pc["uniq_w"], pe["uniq_w"])
    if hasattr(A, "rowptr"):
        assert torch.equal(Y_c, Y_e)                 # CSR SpMM: one thread block per row range, no atomics
    else:
        assert rel(Y_c, Y_e) < 1e-6                  # dense: split-K partial sums by fp32 atomics
    assert rel(Ys_c, Ys_e) < 1e-6 and rel(Gs_c, Gs_e) < 1e-12 and rel(G_c, G_e) < 1e-12
    assert rel(Xl_c, Xl_e) < 1e-6 and rel(Xe_c, Xe_e) < 1e-6


@pytest.mark.parametrize("mode", ["exact", "lvs"])
def test_two_solvers_on_two_streams(mode):
    """Solvers on different data, advanced alternately on two streams, equal each solver run
    alone (1 iteration for LvS: its later plans follow fp32 scores whose last bits depend on the
    atomics' order)."""
    iters = 4 if mode == "exact" else 1
    runs = []
    for seed in (1, 2):
        d = make_input("c2", seed=seed, n_override=20_000)
        runs.append((S.DeviceMatrix.from_host(d["A"]), d["H0"], d["alpha"], d["cfg"]))
    kw = lambda cfg: dict(s=cfg.s, tau=cfg.tau, seed=cfg.seed) if mode == "lvs" else {}
    alone = []
    for M, H0, alpha, cfg in runs:
        W, H = cu(H0), cu(H0)
        sv = S.Solver(M, W, H, alpha, mode=mode, max_iters=iters, **kw(cfg))
        sv.run(iters)
        assert sv.stats()["status"] == 0
        sv.close()
        alone.append((W, H))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    both, solvers = [], []
    for (M, H0, alpha, cfg), st in zip(runs, streams):
        with torch.cuda.stream(st):
            W, H = cu(H0), cu(H0)
            solvers.append(S.Solver(M, W, H, alpha, mode=mode, max_iters=iters, **kw(cfg)))
            both.append((W, H))
    for _ in range(iters):
        for sv, st in zip(solvers, streams):
            with torch.cuda.stream(st):
                sv.run(1)
    torch.cuda.synchronize()
    for sv, st in zip(solvers, streams):
        with torch.cuda.stream(st):
            assert sv.stats()["status"] == 0
            sv.close()
    for (Wa, Ha), (Wb, Hb) in zip(alone, both):
        assert rel(Wb, Wa) < 1e-6 and rel(Hb, Ha) < 1e-6


@pytest.mark.parametrize("defect", ["unsorted", "duplicate", "out_of_range"])
def test_solver_rejects_malformed_csr(defect):
    """symnmf.h "CSR inputs": every sparse path searches sorted rows (the column cuts of the EXACT
    tile passes, the destination ranges of the sampled scatter), so solver creation checks each
    row's columns on the device and returns SYMNMF_ERR_ARG instead of silently misrouting."""
    from synth.configs import CsrMatrix
    d = make_input("c2", n_override=4_000)
    A, H0, alpha = d["A"], d["H0"], d["alpha"]
    col = A.colidx.copy()
    r = int(np.argmax(np.diff(A.rowptr) >= 3))
    s0 = int(A.rowptr[r])
    if defect == "unsorted":
        col[s0], col[s0 + 1] = col[s0 + 1], col[s0]
    elif defect == "duplicate":
        col[s0 + 1] = col[s0]
    else:
        col[s0 + 2] = A.n
    B = CsrMatrix(A.n, A.rowptr, col, A.val)
    M = S.DeviceMatrix.from_host(B)
    for mode, kw in (("exact", {}), ("lvs", dict(s=200, tau=1.0 / 200, seed=1))):
        with pytest.raises(S.A.SymNMFError):
            S.Solver(M, cu(H0), cu(H0), alpha, mode=mode, max_iters=1, **kw)
    # the well-formed matrix is accepted
    sv = S.Solver(S.DeviceMatrix.from_host(A), cu(H0), cu(H0), alpha, mode="exact", max_iters=1)
    sv.close()

