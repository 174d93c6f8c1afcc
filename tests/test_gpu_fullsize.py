"""GPU parity at BASELINE.json's full sizes (c3, c4, c5), in the configuration bench.py times,
on sampled outputs the fp64 oracle computes one by one.

Every checked quantity is row-local given small global ones the oracle forms exactly:
  * a row of A F                 -- row r of A times F, fp64
  * a leverage score (Eq. 2.10)   -- f_r G^{-1} f_r^T with G = F^T F in fp64
  * the hybrid plan          -- bit-exact from the GPU's fp32 scores (Z6)
  * a row of the sampled product Y_s     -- sum over U of omega_u A[U_u, c] f_u
  * a row of the first half's sweep      -- Eq. 2.6 on row r with G, Y[r], F[r], X[r]
EXACT/LAI: the solver runs one full iteration; W after it is the W-half's output (the H-half does
not touch W), so rows of W are checked against the oracle sweep of those rows.
LvS: after one solver iteration, the scores and plan the solver drew for its H-half (side 1,
F = W1) are read back (symnmf_solver_last_plan); the scores are checked on sampled rows, the plan
bit-exactly against the oracle sampler fed those scores, and rows of H1 against the oracle sweep
with G_s and rows of Y_s formed in fp64 from that plan.
Tolerances: 1e-5 relative (Frobenius over the sampled rows) for products, scores and sweeps in
fp32 and in 3xTF32 alike (the 3xTF32 GEMM drains its tensor-core accumulator every 16 k-blocks,
which keeps the truncation bias of the fp32 accumulate near 1e-6 at n = 30,000; tc_gemm.cu).
"""
import numpy as np
import pytest

import oracle as O
from synth import make_input

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2402_08134_b200 import symnmf as S  # noqa: E402

NS = 192   # sampled output rows per check


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def rows_times(A, idx, F, cols=None):
    """A[idx, cols] @ F in fp64, F given for the rows `cols` (all of 0..n-1 when None);
    dense A row by row, CSR A from each row's nonzeros."""
    F = np.asarray(F, dtype=np.float64)
    if not hasattr(A, "rowptr"):
        Ar = np.asarray(A[idx], dtype=np.float64)
        return Ar @ F if cols is None else Ar[:, cols] @ F
    pos = None
    if cols is not None:
        pos = np.full(A.n, -1, dtype=np.int64)
        pos[cols] = np.arange(len(cols))
    out = np.zeros((len(idx), F.shape[1]))
    for t, r in enumerate(idx):
        s, e = A.rowptr[r], A.rowptr[r + 1]
        c, v = A.colidx[s:e].astype(np.int64), A.val[s:e].astype(np.float64)
        if pos is not None:
            p = pos[c]
            c, v = p[p >= 0], v[p >= 0]
        out[t] = v @ F[c]
    return out


def sample_rows(n, seed, tile=None, stride=1):
    """NS random rows, plus (tile given) the first and last row of every `stride`-th tile of `tile`
    rows, every row of the ragged last tile and rows 0 and n - 1: tile boundaries, where a kernel's
    row indexing, carries and masking can go wrong, are always checked."""
    idx = set(np.random.default_rng(seed).choice(n, size=NS, replace=False).tolist()) | {0, n - 1}
    if tile:
        starts = np.arange(0, n, tile)[::stride]
        idx |= set(starts.tolist()) | set(np.minimum(starts + tile - 1, n - 1).tolist())
        idx |= set(range((n - 1) // tile * tile, n))
    return np.array(sorted(idx), dtype=np.int64)


def check_product_scores_plan_sampled(d, precision, seed, tile=None, stride=1):
    A, H0, cfg = d["A"], d["H0"], d["cfg"]
    n, k = cfg.n, cfg.k
    M = S.DeviceMatrix.from_host(A)
    F = cu(H0)
    idx = sample_rows(n, seed, tile, stride)
    # (a10) rows of A F
    Y = S.ah(M, F, precision=precision).cpu().numpy()
    ref = rows_times(A, idx, H0)
    assert rel(Y[idx], ref) < 1e-5      # 3xTF32 too: the GEMM drains its accumulator (tc_gemm.cu)
    # (a1-a3) scores: l_r = f_r G^{-1} f_r^T
    lev = S.leverage_scores(F)
    lg = lev.cpu().numpy()
    G = O.gram(H0)
    Fi = H0[idx].astype(np.float64)
    lref = np.einsum("ij,ij->i", Fi @ np.linalg.inv(G), Fi)
    assert rel(lg[idx], lref) < 1e-5
    assert abs(lg.astype(np.float64).sum() - k) < 1e-3 * k          # sum of scores = rank
    # (a4-a7) the plan, bit-exact from the GPU's fp32 scores
    plan = S.hybrid_sample(lev, k, cfg.s, cfg.tau, seed=cfg.seed, iteration=0, side=0)
    ph = plan.to_host()
    op = O.build_plan(lg, k, cfg.s, cfg.tau, cfg.seed, 0, 0)
    assert np.array_equal(ph["uniq_idx"], op["uniq_idx"]) and np.array_equal(ph["uniq_w"], op["uniq_w"])
    assert (ph["s_D"], ph["s_R"]) == (op["s_D"], op["s_R"])
    # (a8, a9) rows of the sampled product and the sampled Gram
    Ys, Gs = S.sampled_ah(M, F, plan)
    U, w = op["uniq_idx"], op["uniq_w"]
    FU = H0[U].astype(np.float64) * w[:, None]
    Yref = rows_times(A, idx, FU, cols=U)                           # A[c, U] = A[U, c] (symmetry)
    assert rel(Ys.cpu().numpy()[idx], Yref) < 1e-5
    assert rel(Gs.cpu().numpy(), H0[U].astype(np.float64).T @ FU) < 1e-5
    return M, idx


def check_solver_exact_w_rows(d, M, idx, precision, tol):
    """One EXACT solver iteration; rows of W = the oracle sweep (Eq. 2.6) of those rows."""
    A, H0, alpha = d["A"], d["H0"], d["alpha"]
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="exact", precision=precision, max_iters=1)
    sv.run(1)
    assert sv.stats()["status"] == 0
    sv.close()
    Wg = W.cpu().numpy()
    assert np.isfinite(Wg).all() and (Wg >= 0).all()
    Yr = rows_times(A, idx, H0)
    Wr = O.hals_sweep(O.gram(H0), Yr, H0[idx], H0[idx], alpha)
    assert rel(Wg[idx], Wr) < tol


def check_solver_lvs_h_rows(d, M, idx):
    """One LvS solver iteration (as bench.py runs it); the H-half against the oracle."""
    A, H0, alpha, cfg = d["A"], d["H0"], d["alpha"], d["cfg"]
    k = cfg.k
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="lvs", s=cfg.s, tau=cfg.tau, seed=cfg.seed, max_iters=1)
    sv.run(1)
    st = sv.stats()
    assert st["status"] == 0
    lev, plan = sv.last_plan()
    ph = plan.to_host()
    sv.close()
    W1, H1 = W.cpu().numpy(), H.cpu().numpy()
    assert np.isfinite(H1).all() and (H1 >= 0).all()
    lg = lev.cpu().numpy()
    F = W1.astype(np.float64)
    lref = np.einsum("ij,ij->i", F[idx] @ np.linalg.inv(F.T @ F), F[idx])
    assert rel(lg[idx], lref) < 1e-5
    op = O.build_plan(lg, k, cfg.s, cfg.tau, cfg.seed, 0, 1)
    assert (ph["s_D"], ph["s_R"], ph["n_uniq"]) == (op["s_D"], op["s_R"], len(op["uniq_idx"]))
    assert (ph["s_D"], ph["s_R"], ph["n_uniq"]) == tuple(st["halves"][1][x] for x in ("s_D", "s_R", "n_uniq"))
    assert np.array_equal(ph["uniq_idx"], op["uniq_idx"]) and np.array_equal(ph["uniq_w"], op["uniq_w"])
    U, w = op["uniq_idx"], op["uniq_w"]
    FU = F[U] * w[:, None]
    Gs = F[U].T @ FU
    Ys = rows_times(A, idx, FU, cols=U)                             # A[c, U] = A[U, c] (symmetry)
    Hr = O.hals_sweep(Gs, Ys, W1[idx], H0[idx], alpha)
    assert rel(H1[idx], Hr) < 1e-5


@pytest.fixture(scope="module")
def c3():
    return make_input("c3")


@pytest.fixture(scope="module")
def c4():
    return make_input("c4")


def test_c3_full_size_sampled_parity(c3):
    """c3 (dense n = 30,000, k = 32): 3xTF32 product rows, scores, plan, sampled-product rows,
    and W rows after one EXACT solver iteration (3xTF32, as bench.py times it)."""
    M, idx = check_product_scores_plan_sampled(c3, "3xtf32", seed=31, tile=128)
    check_solver_exact_w_rows(c3, M, idx, "3xtf32", 1e-5)


def test_c3_full_size_lvs_solver_half_vs_oracle(c3):
    """c3 LvS (s = 3,000): the solver's scores, plan and H rows after one iteration."""
    M = S.DeviceMatrix.from_host(c3["A"])
    check_solver_lvs_h_rows(c3, M, sample_rows(c3["cfg"].n, 32, tile=256))


def test_c4_full_size_sampled_parity(c4):
    """c4 (CSR n = 2,000,000, 1e8 nonzeros, k = 32): SpMM rows, scores, plan (s = 20,000, with a
    non-empty deterministic set), sampled-product rows, and W rows after one EXACT solver
    iteration (the nnz-balanced SpMM + streaming sweep, as bench.py times it)."""
    M, idx = check_product_scores_plan_sampled(c4, "fp32", seed=41, tile=256, stride=7)
    check_solver_exact_w_rows(c4, M, idx, "fp32", 1e-5)


def test_c4_full_size_lvs_solver_half_vs_oracle(c4):
    """c4 LvS (s = 20,000, hub rows in the deterministic set): the solver's scores, plan and H
    rows after one iteration (destination-range scatter passes, fused Gram, as bench.py runs)."""
    M = S.DeviceMatrix.from_host(c4["A"])
    check_solver_lvs_h_rows(c4, M, sample_rows(c4["cfg"].n, 42, tile=256, stride=7))


def test_c5_full_size_lai_sampled_parity():
    """c5 (dense n = 60,000, 14.4 GB, LAI l = 74, q = 2, k = 64): the range finder's U is
    orthonormal with |lambda| descending, and W rows after one fused LAI iteration equal the oracle
    sweep of those rows with Y[r] = U[r] (Lambda (U^T H0)) formed in fp64 from the same U, Lambda."""
    d = make_input("c5")
    A, H0, alpha, cfg = d["A"], d["H0"], d["alpha"], d["cfg"]
    M = S.DeviceMatrix.from_host(A)
    del A
    U, lam = S.rangefinder(M, cfg.l, cfg.q, cfg.seed, precision="3xtf32")
    Ug, lg = U.cpu().numpy().astype(np.float64), lam.cpu().numpy()
    assert np.abs(Ug.T @ Ug - np.eye(cfg.l)).max() < 1e-4
    assert (np.diff(np.abs(lg)) <= 1e-12 * np.abs(lg).max()).all()
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="lai", precision="3xtf32", max_iters=1, U=U, lam=lam)
    sv.run(1)
    assert sv.stats()["status"] == 0
    sv.close()
    idx = sample_rows(cfg.n, 51, tile=128)
    H64 = H0.astype(np.float64)
    G = H64.T @ H64
    Mx = lg[:, None] * (Ug.T @ H64)                                 # Lambda U^T H0
    Yr = Ug[idx] @ Mx
    Wr = O.hals_sweep(G, Yr, H0[idx], H0[idx], alpha)
    assert rel(W.cpu().numpy()[idx], Wr) < 1e-4


def test_3xtf32_gemm_has_no_accumulation_drift():
    """The tensor core's fp32 accumulate truncates; a K range accumulated in one TMEM chain drifts
    low in proportion to its length (measured -2.1e-4 at n = 30,000 before the drain).  Uniform
    positive data (no cancellation) at c3's size: the signed mean error on sampled rows stays at
    the fp32 level."""
    n, k = 30_016, 32
    rng = np.random.default_rng(7)
    A = rng.random((n, n), dtype=np.float32)
    A = (A + A.T) * np.float32(0.5)
    X = rng.random((n, k), dtype=np.float32)
    Y = S.ah(S.DeviceMatrix.from_host(A), cu(X), precision="3xtf32").cpu().numpy()
    idx = sample_rows(n, 71)
    ref = A[idx].astype(np.float64) @ X.astype(np.float64)
    e = (Y[idx] - ref) / ref
    assert abs(e.mean()) < 5e-6 and np.abs(e).max() < 1e-5


# ------------------------------------------------------------------ 10 iterations at full size
ITERS = 10


def residual_parity(A, Hg, Hr):
    """North star: normalised residual ||A - H H^T||_F / ||A||_F within 1e-4 relative after 10
    iterations."""
    rg, ro = O.residual(A, Hg), O.residual(A, Hr)
    assert abs(rg - ro) <= 1e-4 * ro, (rg, ro)
    return rg, ro


def run_exact(d, M, precision):
    A, H0, alpha = d["A"], d["H0"], d["alpha"]
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="exact", precision=precision, max_iters=ITERS)
    sv.run(ITERS)
    assert sv.stats()["status"] == 0
    sv.close()
    _, Hr, _ = O.iterate(A, H0, H0, alpha, ITERS, "exact")
    return residual_parity(A, H.cpu().numpy(), Hr)


def run_lvs_recorded(d, M):
    """The solver path bench.py times, free-running for 10 iterations with every half's scores and
    plan recorded (SYMNMF_RECORD_PLANS); each plan is checked bit-exactly against the oracle sampler
    fed the GPU's scores of that half (Z6), then the oracle replays those plans in fp64 (O-11
    replay mode) and the residuals after 10 iterations are compared."""
    A, H0, alpha, cfg = d["A"], d["H0"], d["alpha"], d["cfg"]
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="lvs", s=cfg.s, tau=cfg.tau, seed=cfg.seed, max_iters=ITERS,
                  record_plans=True)
    sv.run(ITERS)
    st = sv.stats()
    assert st["status"] == 0
    plans = {}
    for t in range(ITERS):
        for side in (0, 1):
            lev, plan = sv.plan_history(t, side)
            ph, lg = plan.to_host(), lev.cpu().numpy()
            op = O.build_plan(lg, cfg.k, cfg.s, cfg.tau, cfg.seed, t, side)
            assert (ph["s_D"], ph["s_R"], ph["n_uniq"]) == (op["s_D"], op["s_R"], op["n_uniq"]), (t, side)
            assert np.array_equal(ph["uniq_idx"], op["uniq_idx"]) and np.array_equal(ph["uniq_w"], op["uniq_w"])
            assert abs(lg.astype(np.float64).sum() - cfg.k) < 1e-3 * cfg.k            # sum of scores = rank
            plans[(t, side)] = op
    sv.close()
    _, Hr, _ = O.iterate(A, H0, H0, alpha, ITERS, "lvs", s=cfg.s, tau=cfg.tau, seed=cfg.seed, plans=plans)
    return residual_parity(A, H.cpu().numpy(), Hr)


def test_c3_full_size_10_iterations_exact_3xtf32(c3):
    """c3 EXACT with the 3xTF32 tensor-core product, 10 free-running iterations vs fp64."""
    run_exact(c3, S.DeviceMatrix.from_host(c3["A"]), "3xtf32")


def test_c3_full_size_10_iterations_lvs(c3):
    """c3 LvS (s = 3,000), 10 iterations, every plan bit-exact, residual vs the replaying oracle."""
    run_lvs_recorded(c3, S.DeviceMatrix.from_host(c3["A"]))


def test_c4_full_size_10_iterations_exact(c4):
    """c4 EXACT (nnz-balanced SpMM + streaming sweep, as bench.py times it), 10 iterations."""
    run_exact(c4, S.DeviceMatrix.from_host(c4["A"]), "fp32")


def test_c4_full_size_10_iterations_lvs(c4):
    """c4 LvS (s = 20,000 with a non-empty deterministic set), 10 iterations, as bench.py runs it."""
    run_lvs_recorded(c4, S.DeviceMatrix.from_host(c4["A"]))


@pytest.fixture(scope="module")
def c5():
    return make_input("c5")


def test_c5_full_size_operator_and_10_lai_iterations(c5):
    """c5 (n = 60,000, 14.4 GB): (1) the range finder's operator U Lambda U^T applied to a seeded
    probe block equals the fp64 oracle's Alg. RRF + Apx-EVD operator on the same Omega
    (U is unique only up to rotations in eigenvalue clusters, reading Z29, so operators are compared);
    (2) 10 LAI iterations on the GPU's U, Lambda vs the oracle's LAI iterations on the same U, Lambda:
    residual against the full A within 1e-4 relative."""
    A, H0, alpha, cfg = c5["A"], c5["H0"], c5["alpha"], c5["cfg"]
    M = S.DeviceMatrix.from_host(A)
    U, lam = S.rangefinder(M, cfg.l, cfg.q, cfg.seed, precision="3xtf32")
    Ug, lg = U.cpu().numpy().astype(np.float64), lam.cpu().numpy()
    Uo, lo, _ = O.rangefinder(A, cfg.l, cfg.q, cfg.seed)
    P = np.random.default_rng(55).standard_normal((cfg.n, 8))
    opg = Ug @ (lg[:, None] * (Ug.T @ P))
    opo = Uo @ (lo[:, None] * (Uo.T @ P))
    err = rel(opg, opo)
    print(f"c5 operator rel err {err:.3e}, lambda rel err {rel(lg, lo):.3e}")
    # fp32 storage of the basis between passes (2^-24) and the 3xTF32 products (~1e-6 relative)
    # perturb the captured subspace; the operator difference stays at the 1e-6 level
    assert err < 2e-5 and rel(lg, lo) < 2e-5
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="lai", precision="3xtf32", max_iters=ITERS, U=U, lam=lam)
    sv.run(ITERS)
    assert sv.stats()["status"] == 0
    sv.close()
    _, Hr, _ = O.iterate(A, H0, H0, alpha, ITERS, "lai", U=Ug, lam=lg)
    residual_parity(A, H.cpu().numpy(), Hr)
