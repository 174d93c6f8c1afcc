"""GPU parity: every C-ABI operation vs the fp64 oracle on the same seeded inputs.

Tolerances (north star): products / Grams / sampled products
1e-5 relative Frobenius (fp32 path); scores 1e-5 relative 2-norm (Z21);
plans bit-exact given the same fp32 score vector and (seed, iteration, side);
normalised residual after 10 iterations 1e-4 relative.
"""
import math

import os

import numpy as np
import pytest

import oracle as O
from synth import make_input, random_factor, planted_dense

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2402_08134_b200 import symnmf as S  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def sym_dense(n, seed):
    r = np.random.default_rng(seed)
    X = r.random((n, n))
    return ((X + X.T) / 2).astype(np.float32)


@pytest.fixture(scope="module")
def c1():
    return make_input("c1")


@pytest.fixture(scope="module")
def c2small():
    return make_input("c2", n_override=20_000)


# ------------------------------------------------------------------ (a1) Gram
@pytest.mark.parametrize("n,k", [(1, 1), (7, 3), (1000, 8), (1003, 16), (40_000, 32), (5_001, 64), (100_003, 5)])
def test_gram(n, k):
    F = random_factor(n, k, 1)
    G = S.gram(cu(F)).cpu().numpy()
    ref = O.gram(F)
    assert rel(G, ref) < 1e-6
    assert np.array_equal(G, G.T)


# ------------------------------------------------------------------ (a10) exact product
@pytest.mark.parametrize("n,k", [(1000, 8), (1003, 5), (257, 16), (2048, 32), (300, 64), (5, 1)])
def test_ah_dense_fp32(n, k):
    A = sym_dense(n, n + k)
    F = random_factor(n, k, 2)
    Y = S.ah(S.DeviceMatrix.from_host(A), cu(F)).cpu().numpy()
    assert rel(Y, O.ah(A, F)) < 1e-5


@pytest.mark.parametrize("k", [1, 3, 8, 16, 32, 64])
def test_ah_csr(c2small, k):
    A = c2small["A"]
    F = random_factor(A.n, k, 3)
    Y = S.ah(S.DeviceMatrix.from_host(A), cu(F)).cpu().numpy()
    assert rel(Y, O.ah(A, F)) < 1e-5


def test_ah_dense_equals_csr_storage(c2small):
    sub = make_input("c2", n_override=3_200)["A"]
    F = random_factor(sub.n, 8, 4)
    Yc = S.ah(S.DeviceMatrix.from_host(sub), cu(F)).cpu().numpy()
    Yd = S.ah(S.DeviceMatrix.from_host(sub.to_dense()), cu(F)).cpu().numpy()
    assert rel(Yc, Yd) < 1e-6


# ------------------------------------------------------------------ (a3) scores
@pytest.mark.parametrize("n,k", [(7, 3), (1000, 8), (1003, 16), (50_000, 32), (4_099, 64), (100_000, 1)])
def test_leverage_scores(n, k):
    F = random_factor(n, k, 5)
    lev, G = S.leverage_scores(cu(F), return_gram=True)
    lev = lev.cpu().numpy()
    ref = O.leverage_scores(F)
    assert rel(lev, ref) < 1e-5                                    # Z21 norm-wise
    big = ref >= k / n
    assert np.max(np.abs(lev[big] - ref[big]) / ref[big]) < 1e-4
    assert abs(lev.astype(np.float64).sum() - k) < 1e-4 * k        # sum = rank
    assert rel(G.cpu().numpy(), O.gram(F)) < 1e-6


def test_leverage_scores_closed_forms():
    F = np.zeros((5, 2), np.float32); F[0, 0] = 1; F[1, 1] = 1   # [I2; 0] -> (1, 1, 0, ...)
    lev = S.leverage_scores(cu(F)).cpu().numpy()
    assert np.allclose(lev, [1, 1, 0, 0, 0], atol=1e-6)
    lev = S.leverage_scores(cu(np.ones((64, 1), np.float32))).cpu().numpy()
    assert np.allclose(lev, 1 / 64, rtol=1e-6)


def test_leverage_rank_deficient_uses_jitter():
    F = random_factor(500, 4, 6)
    F[:, 3] = 0.0                                                 # zero column: G singular -> one jitter retry
    lev = S.leverage_scores(cu(F)).cpu().numpy()
    assert abs(lev.sum() - 3) < 1e-3


def test_leverage_not_pd_reported():
    F = np.zeros((100, 3), np.float32)                            # tr(G) = 0: no jitter possible
    with pytest.raises(S.A.SymNMFError) as e:
        S.leverage_scores(cu(F))
    assert e.value.code == S.A.ERR_NOT_PD


# ------------------------------------------------------------------ (a4-a7) plan, bit-exact
def _scores(n, k, seed, power=3):
    F = random_factor(n, k, seed) ** power
    return O.leverage_scores(F).astype(np.float32)


@pytest.mark.parametrize("n,k,s,tau,seed,it,side", [
    (1000, 8, 200, 1 / 200, 0, 0, 0),
    (1000, 8, 200, 1 / 200, 0, 7, 1),
    (100_000, 16, 2000, 1 / 2000, 3, 2, 0),
    (100_000, 16, 2000, 1.0, 3, 2, 1),       # tau = 1: pure i.i.d. sampling
    (7, 3, 5, 1 / 5, 1, 0, 0),
    (1, 1, 1, 1.0, 0, 0, 0),
    (2_000_000, 32, 20_000, 1 / 20_000, 0, 1, 1),
    ((1 << 20) + 17, 4, 30_000, 1 / 30_000, 9, 5, 0),
    (6_500_003, 4, 20_000, 1 / 20_000, 2, 3, 1),   # > 6144 prefix blocks: the one-level draw search
])
def test_hybrid_plan_bit_exact(n, k, s, tau, seed, it, side):
    lev = _scores(n, k, seed + 11)
    g = S.hybrid_sample(cu(lev), k, s, tau, seed, it, side).to_host()
    o = O.build_plan(lev, k, s, tau, seed, it, side)
    assert g["s_D"] == o["s_D"] and g["s_R"] == o["s_R"] and g["n_uniq"] == o["n_uniq"] and g["W"] == o["W"]
    assert np.array_equal(g["det_idx"], o["det_idx"])
    assert np.array_equal(g["draw_idx"], o["draw_idx"])
    assert np.array_equal(g["uniq_idx"], o["uniq_idx"])
    assert np.array_equal(g["uniq_w"], o["uniq_w"])                 # IEEE fp64, fixed op order
    assert abs(g["theta"] - o["theta"]) <= 1e-12 * max(1.0, o["theta"])
    assert abs(g["theta"] + g["xi"] - k) < 1e-12 * k


def test_hybrid_plan_all_deterministic_and_zero_mass():
    lev = _scores(3000, 4, 21)
    tau = float(lev.min()) / 4 * 0.5                              # every row in I_D, needs cap = n
    g = S.hybrid_sample(cu(lev), 4, 10, tau, 0, 0, 0).to_host()
    assert g["s_D"] == 3000 and g["s_R"] == 0 and np.array_equal(g["uniq_idx"], np.arange(3000))
    lev = np.zeros(12, np.float32); lev[:2] = 1.0                 # W = 0 -> s_R = 0
    g = S.hybrid_sample(cu(lev), 2, 10, 0.4, 0, 0, 0).to_host()
    assert g["det_idx"].tolist() == [0, 1] and g["s_R"] == 0 and g["theta"] == 2.0


def test_hybrid_capacity_error():
    lev = _scores(3000, 4, 22)
    with pytest.raises(S.A.SymNMFError) as e:
        S.hybrid_sample(cu(lev), 4, 10, float(lev.min()) / 8, 0, 0, 0, cap=100)
    assert e.value.code == S.A.ERR_CAPACITY


# ------------------------------------------------------------------ (a8, a9) sampled products
def _plan_for(F, k, s, tau, seed=0, it=0, side=0):
    """Both sides sample from the same score vector, computed by the oracle (fp32-rounded)."""
    lev = O.leverage_scores(F).astype(np.float32)
    plan = S.hybrid_sample(cu(lev), k, s, tau, seed, it, side)
    return plan, O.build_plan(lev, k, s, tau, seed, it, side)


def test_sampled_dense(c1):
    A, cfg = c1["A"], c1["cfg"]
    F = c1["H0"]
    plan, o = _plan_for(F, cfg.k, cfg.s, cfg.tau)
    Y, Gs = S.sampled_ah(S.DeviceMatrix.from_host(A), cu(F), plan)
    Gr, Yr = O.sampled_products(A, F, o["uniq_idx"], o["uniq_w"])
    assert rel(Y.cpu().numpy(), Yr) < 1e-5 and rel(Gs.cpu().numpy(), Gr) < 1e-6


@pytest.mark.parametrize("n,k,s", [(1000, 8, 200), (3000, 32, 1500), (4100, 16, 900), (2052, 64, 700),
                                   (1998, 32, 300), (5000, 3, 2000), (640, 32, 10), (12_000, 32, 3000)])
@pytest.mark.parametrize("path", ["tc", "simt"])
def test_sampled_dense_paths(n, k, s, path, monkeypatch):
    """Sampled dense product Y_s = A[U,:]^T (Omega F[U]): the tcgen05 3xTF32 kernel
    (tc_sampled.cu, SYMNMF_SAMPLED_DENSE=tc; the default from n = 16384 when n % 4 == 0, k <= 64) and
    the fp32 SIMT kernel (=simt) vs the oracle.  Ragged output tiles (n % 128 != 0), n % 4 != 0 (SIMT fallback), |U| from
    < 32 (one partial k-block) to the c3 budget (s = 3,000: U split over the grid)."""
    monkeypatch.setenv("SYMNMF_SAMPLED_DENSE", path)
    A = sym_dense(n, n + 7 * k)
    F = random_factor(n, k, 11) ** 2
    plan, o = _plan_for(F, k, s, 1.0 / s, seed=3, it=1, side=0)
    Y, Gs = S.sampled_ah(S.DeviceMatrix.from_host(A), cu(F), plan)
    Gr, Yr = O.sampled_products(A, F, o["uniq_idx"], o["uniq_w"])
    assert rel(Y.cpu().numpy(), Yr) < 1e-5 and rel(Gs.cpu().numpy(), Gr) < 1e-6


def test_sampled_dense_all_rows_equals_exact():
    """Every row deterministic (tau below every p_i): U = all n rows, Omega = 1, so the tensor-core
    sampled product is A F (P:716-719 with I_D = all rows)."""
    n, k = 2_500, 16
    os.environ["SYMNMF_SAMPLED_DENSE"] = "tc"
    A = sym_dense(n, 5)
    F = random_factor(n, k, 12)
    lev = S.leverage_scores(cu(F))
    tau = float(lev.min().item()) / k * 0.5
    plan = S.hybrid_sample(lev, k, 10, tau, 0, 0, 0)
    Y, _ = S.sampled_ah(S.DeviceMatrix.from_host(A), cu(F), plan)
    os.environ.pop("SYMNMF_SAMPLED_DENSE")
    assert plan.to_host()["n_uniq"] == n
    assert rel(Y.cpu().numpy(), O.ah(A, F)) < 1e-5


@pytest.mark.parametrize("shfl", [False, True])
@pytest.mark.parametrize("k", [3, 16, 32, 64])
def test_sampled_csr(c2small, k, shfl, monkeypatch):
    monkeypatch.setenv("SYMNMF_SCATTER_SHFL", "1" if shfl else "0")
    A = c2small["A"]
    F = random_factor(A.n, k, 9) ** 2
    plan, o = _plan_for(F, k, 1000, 1 / 1000, seed=5, it=3, side=1)
    Y, Gs = S.sampled_ah(S.DeviceMatrix.from_host(A), cu(F), plan)
    Gr, Yr = O.sampled_products(A, F, o["uniq_idx"], o["uniq_w"])
    assert rel(Y.cpu().numpy(), Yr) < 1e-5 and rel(Gs.cpu().numpy(), Gr) < 1e-6


def test_sampled_all_rows_equals_exact(c2small):
    A = make_input("c2", n_override=4_000)["A"]
    F = random_factor(A.n, 8, 10)
    lev = S.leverage_scores(cu(F))
    tau = float(lev.min().item()) / 8 * 0.5
    plan = S.hybrid_sample(lev, 8, 10, tau, 0, 0, 0)
    M = S.DeviceMatrix.from_host(A)
    Y, Gs = S.sampled_ah(M, cu(F), plan)
    assert rel(Y.cpu().numpy(), S.ah(M, cu(F)).cpu().numpy()) < 1e-6
    assert rel(Gs.cpu().numpy(), O.gram(F)) < 1e-6


# ------------------------------------------------------------------ (a11) HALS sweep
@pytest.mark.parametrize("n,k", [(1000, 8), (1001, 5), (20_000, 16), (3_000, 32), (777, 64)])
def test_hals_sweep(n, k):
    r = np.random.default_rng(n + k)
    A = sym_dense(min(n, 1500), 7) if n <= 1500 else None
    F = random_factor(n, k, 11)
    X = random_factor(n, k, 12)
    G = O.gram(F)
    Y = (A @ F.astype(np.float64)).astype(np.float32) if A is not None else \
        (F.astype(np.float64) @ G + r.random((n, k))).astype(np.float32)
    alpha = 0.7
    Xg, Gn = S.hals_sweep(cu(G), cu(Y), cu(F), cu(X), alpha, return_gram=True)
    Xr = O.hals_sweep(G, Y, F, X, alpha)
    assert rel(Xg.cpu().numpy(), Xr) < 1e-5
    assert rel(Gn.cpu().numpy(), O.gram(Xr)) < 1e-5


def test_hals_fixed_point():
    H = random_factor(500, 6, 13)
    A = (H.astype(np.float64) @ H.T).astype(np.float32)
    G = O.gram(H)
    Y = (A.astype(np.float64) @ H).astype(np.float32)
    X = S.hals_sweep(cu(G), cu(Y), cu(H), cu(H.copy()), 1.3).cpu().numpy()
    assert rel(X, H) < 1e-5


# ------------------------------------------------------------------ (a12, a13) LAI
def test_gaussian_omega_matches_oracle():
    Om = S.gaussian(1001, 13, seed=5).cpu().numpy()
    ref = O.gaussian_omega(1001, 13, seed=5)
    assert np.max(np.abs(Om - ref)) <= 2e-6 * max(1.0, np.abs(ref).max())
    assert np.mean(Om == ref) > 0.999


def test_lai_apply():
    r = np.random.default_rng(3)
    U = np.linalg.qr(r.standard_normal((3000, 20)))[0].astype(np.float32)
    lam = r.standard_normal(20) * 10
    F = random_factor(3000, 16, 14)
    Y = S.lai_ah(cu(U), cu(lam), cu(F)).cpu().numpy()
    assert rel(Y, O.lai_apply(U, lam, F)) < 1e-5


def test_rangefinder_low_rank_exact():
    r = np.random.default_rng(4)
    n, rank, l = 1200, 10, 16
    B = r.standard_normal((n, rank))
    A = (B @ np.diag(np.linspace(1, 10, rank)) @ B.T).astype(np.float32)
    U, lam = S.rangefinder(S.DeviceMatrix.from_host(A), l, 2, seed=1)
    U, lam = U.cpu().numpy().astype(np.float64), lam.cpu().numpy()
    assert np.allclose(U.T @ U, np.eye(l), atol=1e-5)
    Ar = U @ np.diag(lam) @ U.T
    assert rel(Ar, A) < 1e-5                                        # exact-rank capture
    Uo, lo, _ = O.rangefinder(A, l, 2, seed=1)
    assert np.allclose(np.sort(np.abs(lam))[-rank:], np.sort(np.abs(lo))[-rank:], rtol=1e-5)


def test_rangefinder_gaussian_kernel_operator():
    d = make_input("c3", n_override=2_000)
    A = d["A"]
    l = 40
    U, lam = S.rangefinder(S.DeviceMatrix.from_host(A), l, 2, seed=0)
    Uo, lo, _ = O.rangefinder(A, l, 2, seed=0)
    P = random_factor(A.shape[0], 8, 15)
    Yg = O.lai_apply(U.cpu().numpy(), lam.cpu().numpy(), P)
    Yo = O.lai_apply(Uo, lo, P)
    # both approximate A to the same accuracy; the operators agree to the tail mass
    assert rel(Yg, Yo) < 2e-4
    assert abs(np.abs(lam.cpu().numpy()[0]) - np.abs(lo[0])) < 1e-5 * abs(lo[0])


# ------------------------------------------------------------------ (a15) residual
def test_residual_dense_and_csr(c1, c2small):
    A, H = c1["A"], c1["H0"]
    out = S.residual(S.DeviceMatrix.from_host(A), cu(H)).cpu().numpy()
    assert abs(out[0] - O.residual(A, H)) < 1e-9
    B = c2small["A"]
    Hb = random_factor(B.n, 16, 16) * 0.05
    out = S.residual(S.DeviceMatrix.from_host(B), cu(Hb)).cpu().numpy()
    assert abs(out[0] - O.residual(B, Hb)) < 1e-7


# ------------------------------------------------------------------ (a14) iterate
def _run(d, mode, iters, **kw):
    A, H0, alpha = d["A"], d["H0"], d["alpha"]
    M = S.DeviceMatrix.from_host(A)
    W, H = cu(H0), cu(H0)
    out = S.iterate(M, W, H, alpha, iters, mode=mode, **kw)
    return W.cpu().numpy(), H.cpu().numpy(), out


def test_iterate_exact_c1(c1):
    _, Hg, out = _run(c1, "exact", 10, with_residual=True)
    _, Hr, _ = O.iterate(c1["A"], c1["H0"], c1["H0"], c1["alpha"], 10, "exact")
    rg, ro = O.residual(c1["A"], Hg), O.residual(c1["A"], Hr)
    assert abs(rg - ro) <= 1e-4 * ro
    assert abs(out["residual"][-1] - rg) < 1e-6


def test_iterate_lvs_c1(c1):
    cfg = c1["cfg"]
    _, Hg, out = _run(c1, "lvs", 10, s=cfg.s, tau=cfg.tau, seed=0)
    _, Hr, tr = O.iterate(c1["A"], c1["H0"], c1["H0"], c1["alpha"], 10, "lvs", s=cfg.s, tau=cfg.tau, seed=0)
    for g, o in zip(out["halves"], tr):
        assert (g["s_D"], g["s_R"], g["n_uniq"]) == (o["s_D"], o["s_R"], o["n_uniq"])
    rg, ro = O.residual(c1["A"], Hg), O.residual(c1["A"], Hr)
    assert abs(rg - ro) <= 1e-4 * ro


@pytest.fixture(scope="module")
def c2():
    return make_input("c2")


def test_iterate_exact_c2(c2):
    _, Hg, out = _run(c2, "exact", 10)
    _, Hr, _ = O.iterate(c2["A"], c2["H0"], c2["H0"], c2["alpha"], 10, "exact")
    rg, ro = O.residual(c2["A"], Hg), O.residual(c2["A"], Hr)
    assert abs(rg - ro) <= 1e-4 * ro, (rg, ro)


def test_iterate_lvs_c2_replayed_oracle_plans(c2):
    """LvS parity at 1e-4 with identical sampling decisions: the GPU replays the
    oracle's per-half plans (index sets depend on the scores' last bits, Z29)."""
    A, H0, alpha, cfg = c2["A"], c2["H0"], c2["alpha"], c2["cfg"]
    _, Hr, tr = O.iterate(A, H0, H0, alpha, 10, "lvs", s=cfg.s, tau=cfg.tau, seed=0, record=True)
    M = S.DeviceMatrix.from_host(A)
    Wg, Hg = cu(H0), cu(H0)
    for t in tr:
        pl = t["plan"]
        F, X = (Hg, Wg) if t["side"] == 0 else (Wg, Hg)
        plan = S.plan_from_arrays(pl["uniq_idx"], pl["uniq_w"], pl["s_D"], pl["s_R"], pl["W"])
        Y, Gs = S.sampled_ah(M, F, plan)
        S.hals_sweep(Gs, Y, F, X, alpha)
    rg, ro = O.residual(A, Hg.cpu().numpy()), O.residual(A, Hr)
    assert abs(rg - ro) <= 1e-4 * ro, (rg, ro)


@pytest.mark.parametrize("cfgname", ["c1", "c2"])
def test_solver_lvs_iteration_equals_abi_composition(cfgname, c1, c2):
    """The fused solver iteration equals the composition of the individual ABI calls
    (scores -> plan -> sampled products -> sweep) on the same device data."""
    d = c1 if cfgname == "c1" else c2
    A, H0, alpha, cfg = d["A"], d["H0"], d["alpha"], d["cfg"]
    M = S.DeviceMatrix.from_host(A)
    W1, H1 = cu(H0), cu(H0)
    sv = S.Solver(M, W1, H1, alpha, mode="lvs", s=cfg.s, tau=cfg.tau, seed=0, max_iters=1)
    sv.run(1)
    st = sv.stats()["halves"]
    W2, H2 = cu(H0), cu(H0)
    for side in (0, 1):
        F, X = (H2, W2) if side == 0 else (W2, H2)
        lev = S.leverage_scores(F)
        plan = S.hybrid_sample(lev, cfg.k, cfg.s, cfg.tau, 0, 0, side)
        ph = plan.to_host()
        assert (ph["s_D"], ph["s_R"], ph["n_uniq"]) == (st[side]["s_D"], st[side]["s_R"], st[side]["n_uniq"])
        Y, Gs = S.sampled_ah(M, F, plan)
        S.hals_sweep(Gs, Y, F, X, alpha)
    assert rel(W1.cpu().numpy(), W2.cpu().numpy()) < 1e-5
    assert rel(H1.cpu().numpy(), H2.cpu().numpy()) < 1e-5


def test_iterate_lvs_c2_free_running_statistical(c2):
    """Independent plans (GPU scores vs oracle scores differ in the last bits): only
    statistical agreement is expected -- parity unpinned for free-running LvS."""
    cfg = c2["cfg"]
    _, Hg, out = _run(c2, "lvs", 10, s=cfg.s, tau=cfg.tau, seed=0)
    _, Hr, tr = O.iterate(c2["A"], c2["H0"], c2["H0"], c2["alpha"], 10, "lvs", s=cfg.s, tau=cfg.tau, seed=0)
    rg, ro = O.residual(c2["A"], Hg), O.residual(c2["A"], Hr)
    # LvS-HALS on c2 is noisy iteration to iteration (residual excursions of several %
    # between plans, tools/debug_lvs.py); only a band is asserted here
    assert abs(rg - ro) <= 1e-1 * ro, (rg, ro)
    assert all(h["s_D"] + h["s_R"] == cfg.s for h in out["halves"])
    sd_g = np.mean([h["s_D"] for h in out["halves"]]); sd_o = np.mean([t["s_D"] for t in tr])
    assert abs(sd_g - sd_o) <= 0.1 * max(sd_o, 1)


def test_iterate_lai_c1(c1):
    A = c1["A"]
    M = S.DeviceMatrix.from_host(A)
    U, lam = S.rangefinder(M, 12, 2, seed=0)
    W, H = cu(c1["H0"]), cu(c1["H0"])
    S.iterate(M, W, H, c1["alpha"], 10, mode="lai", U=U, lam=lam)
    _, Hr, _ = O.iterate(A, c1["H0"], c1["H0"], c1["alpha"], 10, "lai", U=U.cpu().numpy(), lam=lam.cpu().numpy())
    rg, ro = O.residual(A, H.cpu().numpy()), O.residual(A, Hr)
    assert abs(rg - ro) <= 1e-4 * ro


def test_solver_first_iter_keys_the_sampler(c1):
    """A resumed run (first_iter = 3) draws from the Philox streams of iteration 3 (bit-reproducible resume)."""
    cfg = c1["cfg"]
    M = S.DeviceMatrix.from_host(c1["A"])
    W, H = cu(c1["H0"]), cu(c1["H0"])
    sv = S.Solver(M, W, H, c1["alpha"], mode="lvs", s=cfg.s, tau=cfg.tau, seed=0, first_iter=3, max_iters=2)
    sv.run(1)
    st = sv.stats()
    assert st["status"] == 0 and st["iters"] == 1
    lev = O.leverage_scores(c1["H0"]).astype(np.float32)
    o = O.build_plan(lev, cfg.k, cfg.s, cfg.tau, 0, 3, 0)           # side 0 samples rows of H0 at it = 3
    g = st["halves"][0]
    assert (g["s_D"], g["s_R"], g["n_uniq"]) == (o["s_D"], o["s_R"], o["n_uniq"])
    sv.run(1)
    assert sv.stats()["iters"] == 2
    sv.close()


# ------------------------------------------------------------------ (a10) tcgen05 3xTF32
@pytest.mark.parametrize("n,k", [(1000, 8), (1024, 16), (2048, 32), (3000, 64), (1500, 17), (4096, 5), (640, 48)])
def test_ah_dense_3xtf32(n, k):
    A = sym_dense(n, 3 * n + k)
    F = random_factor(n, k, 21)
    Y = S.ah(S.DeviceMatrix.from_host(A), cu(F), precision="3xtf32").cpu().numpy()
    err = rel(Y, O.ah(A, F))
    assert err < 2e-4                                               # north star 3xTF32 tolerance
    assert err < 1e-5                                               # what 3xTF32 actually delivers (fp32 class)


def test_ah_dense_3xtf32_planted_and_ragged():
    d = make_input("c1")
    Y = S.ah(S.DeviceMatrix.from_host(d["A"]), cu(d["H0"]), precision="3xtf32").cpu().numpy()
    assert rel(Y, O.ah(d["A"], d["H0"])) < 2e-6
    A = sym_dense(1003, 5)                                          # lda % 4 != 0: no TMA descriptor
    with pytest.raises(S.A.SymNMFError) as e:
        S.ah(S.DeviceMatrix.from_host(A), cu(random_factor(1003, 8, 1)), precision="3xtf32")
    assert e.value.code == S.A.ERR_UNSUPPORTED


def test_rangefinder_3xtf32_matches_fp32():
    d = make_input("c3", n_override=2_000)
    M = S.DeviceMatrix.from_host(d["A"])
    U1, l1 = S.rangefinder(M, 74, 2, seed=0, precision="fp32")       # l = k + 10 of config c5
    U2, l2 = S.rangefinder(M, 74, 2, seed=0, precision="3xtf32")
    P = random_factor(2000, 8, 3)
    Y1 = O.lai_apply(U1.cpu().numpy(), l1.cpu().numpy(), P)
    Y2 = O.lai_apply(U2.cpu().numpy(), l2.cpu().numpy(), P)
    assert rel(Y2, Y1) < 2e-4


def test_iterate_exact_3xtf32_c1():
    d = make_input("c1")
    _, Hg, _ = _run(d, "exact", 10, precision="3xtf32")
    _, Hr, _ = O.iterate(d["A"], d["H0"], d["H0"], d["alpha"], 10, "exact")
    rg, ro = O.residual(d["A"], Hg), O.residual(d["A"], Hr)
    assert abs(rg - ro) <= 1e-4 * ro


# ------------------------------------------------------------------ CSR tile path (product fused into the sweep)
def _csr_case(cfgname, n, k, seed=7):
    from synth.configs import init_factor, mean_entry
    d = make_input(cfgname, n_override=n)
    A = d["A"]
    H0 = init_factor(n, k, mean_entry(A), np.random.default_rng(seed))
    return A, H0, d["alpha"]


@pytest.mark.parametrize("cfgname,n,k", [("c2", 20_000, 16), ("c2", 20_000, 8), ("c4", 40_000, 32),
                                         ("c4", 40_000, 64), ("c4", 40_032, 16), ("c2", 2_000, 32)])
@pytest.mark.parametrize("tile", ["nnz", "rows"])
def test_csr_tile_exact_one_iteration(cfgname, n, k, tile, monkeypatch):
    """Solver EXACT on CSR, both SpMM forms: the nnz-balanced SpMM (chunks of 256 nonzeros with
    carries, default) and the row-group SpMM (SYMNMF_CSR_SPMM=rows), each followed by the streaming
    sweep: W and H after one iteration vs the oracle's fp64 iteration.  Covers ragged last tiles
    (n % 256 != 0), hub rows (power-law c4 recipe) and k = 8..64."""
    monkeypatch.setenv("SYMNMF_CSR_SPMM", tile)
    monkeypatch.setenv("SYMNMF_SWEEP", "stream")
    A, H0, alpha = _csr_case(cfgname, n, k)
    M = S.DeviceMatrix.from_host(A)
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="exact", max_iters=1)
    sv.run(1)
    assert sv.stats()["status"] == 0
    sv.close()
    Wr, Hr, _ = O.iterate(A, H0, H0, alpha, 1, "exact")
    assert rel(W.cpu().numpy(), Wr) < 1e-5
    assert rel(H.cpu().numpy(), Hr) < 1e-5


@pytest.mark.parametrize("cfgname,n,k,s", [("c4", 40_000, 32, 800), ("c2", 20_000, 16, 400), ("c4", 40_000, 8, 2000)])
@pytest.mark.parametrize("slice_mb", ["", "1", "stream", "stream1", "stream_zero", "noshfl", "stream1_noshfl", "stream1_nomerge"])
def test_csr_lvs_solver_equals_abi_composition(cfgname, n, k, s, slice_mb, monkeypatch):
    """Solver LvS on CSR graphs with hubs (vector-atomic scatter of the sampled product, fused Gram)
    equals the composition of the ABI calls on the same device data; slice_mb = 1 forces several
    destination-range passes of the sampled scatter, "stream" the streaming sweep with G and R in
    the constant bank (the default from 2^20 rows), where the scatter accumulates onto the alpha F the
    previous sweep left in Y ("stream1": with several passes; "stream_zero": Y re-zeroed instead,
    SYMNMF_YALPHA=0; "noshfl": the scatter with broadcast entry loads instead of the default
    coalesced, shuffled ones, SYMNMF_SCATTER_SHFL=0, in the solver and the ABI call)."""
    if slice_mb.startswith("stream"):
        monkeypatch.setenv("SYMNMF_SWEEP", "stream")
    if slice_mb in ("1", "stream1", "stream1_noshfl", "stream1_nomerge"):
        monkeypatch.setenv("SYMNMF_SCATTER_SLICE_MB", "1")
    if slice_mb.endswith("noshfl"):
        monkeypatch.setenv("SYMNMF_SCATTER_SHFL", "0")
    if slice_mb.endswith("nomerge"):
        monkeypatch.setenv("SYMNMF_SCATTER_MERGE", "0")
    if slice_mb == "stream_zero":
        monkeypatch.setenv("SYMNMF_YALPHA", "0")
    A, H0, alpha = _csr_case(cfgname, n, k)
    tau = 1.0 / s
    M = S.DeviceMatrix.from_host(A)
    W1, H1 = cu(H0), cu(H0)
    sv = S.Solver(M, W1, H1, alpha, mode="lvs", s=s, tau=tau, seed=3, max_iters=1)
    sv.run(1)
    st = sv.stats()
    assert st["status"] == 0
    sv.close()
    W2, H2 = cu(H0), cu(H0)
    for side in (0, 1):
        F, X = (H2, W2) if side == 0 else (W2, H2)
        lev = S.leverage_scores(F)
        plan = S.hybrid_sample(lev, k, s, tau, 3, 0, side)
        ph = plan.to_host()
        assert (ph["s_D"], ph["s_R"], ph["n_uniq"]) == (st["halves"][side]["s_D"], st["halves"][side]["s_R"],
                                                         st["halves"][side]["n_uniq"])
        Y, Gs = S.sampled_ah(M, F, plan)
        S.hals_sweep(Gs, Y, F, X, alpha)
    assert rel(W1.cpu().numpy(), W2.cpu().numpy()) < 1e-5
    assert rel(H1.cpu().numpy(), H2.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("sweep", ["stream", "fused"])
def test_csr_lvs_replayed_plan_vs_oracle(sweep, monkeypatch):
    """One LvS half through the solver vs the oracle's sampled products + sweep fed the plan the
    GPU drew (the same plan is recomputed by the ABI sampler from the same device scores)."""
    monkeypatch.setenv("SYMNMF_SWEEP", sweep)
    A, H0, alpha = _csr_case("c4", 30_016, 32)
    s, tau = 600, 1.0 / 600
    M = S.DeviceMatrix.from_host(A)
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="lvs", s=s, tau=tau, seed=5, max_iters=1)
    sv.run(1)
    sv.close()
    lev = S.leverage_scores(cu(H0))
    ph = S.hybrid_sample(lev, 32, s, tau, 5, 0, 0).to_host()
    Gs, Ys = O.sampled_products(A, H0, ph["uniq_idx"], ph["uniq_w"])
    Wr = O.hals_sweep(Gs, Ys, H0, H0, alpha)
    assert rel(W.cpu().numpy(), Wr) < 1e-5


@pytest.mark.parametrize("n,l", [(3000, 74), (2_049, 40)])
def test_lai_fused_half_matches_oracle_and_four_kernel_path(n, l, monkeypatch):
    """LAI-SymNMF with k = 64: the fused launch per half (Y = U (Lambda U^T F) per tile, sweep,
    X^T X and Lambda U^T X for the next half) against the four-kernel half and the fp64 oracle
    iterating on the same U, Lambda.  n = 2049 leaves a 1-row last tile."""
    from synth.configs import init_factor
    X = np.random.default_rng(3).random((n, 16))
    A = (X @ X.T / 16).astype(np.float32)
    k = 64
    H0 = init_factor(n, k, float(A.mean()), np.random.default_rng(4))
    alpha = float(A.max())
    M = S.DeviceMatrix.from_host(A)
    U, lam = S.rangefinder(M, l, 1, seed=0)
    res = {}
    for mode in ("auto", "never"):
        if mode == "never":
            monkeypatch.setenv("SYMNMF_LAI_FUSED", "never")
        W, H = cu(H0), cu(H0)
        S.iterate(M, W, H, alpha, 3, mode="lai", U=U, lam=lam)
        res[mode] = (W.cpu().numpy(), H.cpu().numpy())
    _, Hr, _ = O.iterate(A, H0, H0, alpha, 3, "lai", U=U.cpu().numpy(), lam=lam.cpu().numpy())
    assert rel(res["auto"][1], Hr) < 1e-4 and rel(res["never"][1], Hr) < 1e-4
    # the two fp32 paths differ in summation order only (U^T X per tile vs one cross Gram)
    assert rel(res["auto"][1], res["never"][1]) < 5e-5
    assert rel(res["auto"][0], res["never"][0]) < 5e-5


# ------------------------------------------------------------------ NEXT-3 convergence protocol
@pytest.mark.parametrize("which,precision", [("c1", "fp32"), ("c1", "3xtf32"), ("c2small", "fp32")])
def test_projected_gradient_vs_oracle(which, precision, c1, c2small):
    """||P grad f(H)|| and ||grad f(H)|| (App. D) at the initial factor and after two
    HALS iterations (where part of H has hit the bound and the KKT mask matters)."""
    d = c1 if which == "c1" else c2small
    A, H0, alpha = d["A"], d["H0"], d["alpha"]
    M = S.DeviceMatrix.from_host(A)
    tol = 1e-5 if precision == "fp32" else 2e-4
    W, H = cu(H0), cu(H0)
    for it in range(2):
        pg = S.projected_gradient(M, H, precision).cpu().numpy()
        opg, og = O.projected_gradient(A, H.cpu().numpy())
        assert abs(pg[0] - opg) <= tol * opg and abs(pg[1] - og) <= tol * og
        S.iterate(M, W, H, alpha, 2, mode="exact")
    Hn = H.cpu().numpy()
    assert (Hn == 0).any()   # the mask is exercised


@pytest.mark.parametrize("mode", ["exact", "lvs"])
def test_solver_records_projected_gradient(mode, c1):
    """The solver's per-iteration projected-gradient norm (with_residual) equals the oracle's
    formula evaluated on the GPU's own H after each of 4 iterations."""
    A, H0, alpha, cfg = c1["A"], c1["H0"], c1["alpha"], c1["cfg"]
    M = S.DeviceMatrix.from_host(A)
    W, H = cu(H0), cu(H0)
    kw = dict(s=cfg.s, tau=cfg.tau, seed=0) if mode == "lvs" else {}
    sv = S.Solver(M, W, H, alpha, mode=mode, max_iters=4, with_residual=True, **kw)
    pgs = []
    for t in range(4):
        sv.run(1)
        pgs.append(O.projected_gradient(A, H.cpu().numpy())[0])
    got = sv.pgrad()
    assert sv.stats()["status"] == 0
    for g, o in zip(got, pgs):
        assert abs(g - o) <= 1e-5 * o
    sv.close()


def test_run_until_stops_where_the_oracle_stops(c1):
    """P:1086 stopping rule on c1 EXACT: the GPU solver stops after the same number of iterations
    as the oracle's driver (unless a residual decrease lies within 1e-6 of the 1e-4 threshold,
    where fp32 rounding may decide either way)."""
    A, H0, alpha = c1["A"], c1["H0"], c1["alpha"]
    _, _, res, done = O.solve(A, H0, alpha, 300)
    M = S.DeviceMatrix.from_host(A)
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="exact", max_iters=300, with_residual=True)
    ran = sv.run_until(300)
    r_gpu = sv.stats()["residual"]
    sv.close()
    assert len(r_gpu) == ran
    margins = [abs((res[t - 1] - res[t]) - 1e-4) for t in range(1, len(res))]
    if min(margins) > 1e-6:
        assert ran == done
    assert abs(r_gpu[-1] - res[min(ran, len(res)) - 1]) <= 1e-4 * res[-1]
    assert O.stop_index(r_gpu) == ran


# ------------------------------------------------------------------ NEXT-2 Ada-RRF + Iterative Refinement
@pytest.mark.parametrize("precision", ["fp32", "3xtf32"])
def test_adaptive_rangefinder_vs_oracle(precision):
    """Ada-RRF: same number of passes as the oracle (unless a residual decrease lies
    within 1e-5 of the 1e-3 threshold), residual trick values within 1e-5, and the same LAI
    operator U Lambda U^T on a probe block."""
    r = np.random.default_rng(8)
    n = 2048
    X = r.standard_normal((n, 32))
    A = (X @ X.T / 32 + 0.02 * np.eye(n)).astype(np.float32)
    M = S.DeviceMatrix.from_host(A)
    U, lam, passes, res = S.rangefinder_adaptive(M, 40, 8, seed=4, tol=1e-3, precision=precision)
    Uo, lamo, Qo, po, reso = O.rangefinder_adaptive(A, 40, 8, seed=4, tol=1e-3)
    # the trick r^2 = 1 - ||B||^2 / ||A||^2 cancels: a relative bias eps in ||B||^2 moves r by
    # ~eps / (2 r).  B is formed by the fp32 SIMT product in both precisions (reading R3): its
    # round-to-nearest errors are unbiased and cancel in the fp64 sum, so r is held to 0.2% relative
    dr = [2e-3 * b_ for b_ in reso]
    margins = [abs((reso[i] - reso[i + 1]) - 1e-3) - dr[i] - dr[i + 1] for i in range(len(reso) - 1)]
    if not margins or min(margins) > 0:
        assert passes == po
    for a_, b_, d_ in zip(res, reso, dr):
        assert abs(a_ - b_) <= d_
    P = r.standard_normal((n, 6))
    Ug, lg = U.cpu().numpy().astype(np.float64), lam.cpu().numpy()
    got = Ug @ (lg[:, None] * (Ug.T @ P))
    ref = Uo @ (lamo[:, None] * (Uo.T @ P))
    assert rel(got, ref) < (1e-4 if precision == "fp32" else 5e-4)


def test_solve_lai_with_iterative_refinement_vs_oracle(c1):
    """LAI-SymNMF until the P:1086 rule, then Iterative Refinement on the full A: the
    GPU driver ends where the oracle's does (residual within 1e-4 relative; iteration counts
    equal unless a decrease sits within 1e-6 of the rule's 1e-4) and below the LAI phase."""
    A, H0, alpha = c1["A"], c1["H0"], c1["alpha"]
    M = S.DeviceMatrix.from_host(A)
    U, lam = S.rangefinder(M, 4, 1, seed=0)
    W, H = cu(H0), cu(H0)
    out = S.solve(M, W, H, alpha, 200, mode="lai", U=U, lam=lam, refine=True)
    _, _, r1, r2 = O.solve_lai_ir(A, H0, alpha, U.cpu().numpy(), lam.cpu().numpy(), 200)
    g1, g2 = out["residual"]
    assert len(g1) == out["iters"][0] and len(g2) == out["iters"][1]
    near = lambda r: min([abs((r[t - 1] - r[t]) - 1e-4) for t in range(1, len(r))] or [1.0]) <= 1e-6
    if not near(r1) and not near(r2):
        assert out["iters"] == [len(r1), len(r2)]
    assert abs(g2[-1] - r2[-1]) <= 1e-4 * r2[-1]
    assert g2[-1] < g1[-1]
    assert abs(O.residual(A, H.cpu().numpy()) - g2[-1]) <= 1e-5


# ------------------------------------------------------------------ NEXT-1 BPP update
@pytest.mark.parametrize("n,k", [(3000, 8), (2049, 16), (1500, 32), (777, 5), (40, 3), (900, 64), (513, 48)])
def test_bpp_update_vs_oracle(n, k):
    """Exact per-row NLS by block principal pivoting (App. G) vs the fp64 oracle BPP on the
    same (G, Y, F): regularised problems from a random factor, right-hand sides with mixed signs
    so that active sets are non-trivial."""
    r = np.random.default_rng(n + k)
    F = r.random((n, k)).astype(np.float32)
    G = F.astype(np.float64).T @ F.astype(np.float64)
    Y = (r.standard_normal((n, k)) * 3 + 1).astype(np.float32)
    alpha = 0.5
    X = cu(np.zeros((n, k), np.float32))
    Xg, Gn, nc = S.bpp_update(cu(G), cu(Y), cu(F), X, alpha, return_gram=True)
    Xo = O.bpp_update(G, Y, F, alpha)
    assert nc == 0
    assert rel(Xg.cpu().numpy(), Xo) < 1e-6
    # the entry value of X is not used
    Xw = cu((r.random((n, k)) > 0.5).astype(np.float32))
    Xw, nc2 = S.bpp_update(cu(G), cu(Y), cu(F), Xw, alpha)
    assert nc2 == 0 and rel(Xw.cpu().numpy(), Xo) < 1e-6
    assert (Xg.cpu().numpy() == 0).any() and (Xg.cpu().numpy() > 0).any()
    assert rel(Gn.cpu().numpy(), O.gram(Xg.cpu().numpy())) < 1e-6


@pytest.mark.parametrize("mode", ["exact", "lvs"])
def test_solver_bpp_rule_vs_oracle(mode, c1):
    """ANLS-BPP / LvS-BPP iterations through the solver vs the oracle's
    iterate(rule="bpp"): normalised residual after 5 iterations within 1e-4 (LvS: same plans, the
    scores of an exactly solved factor being reproducible to fp32 rounding)."""
    A, H0, alpha, cfg = c1["A"], c1["H0"], c1["alpha"], c1["cfg"]
    kw = dict(s=cfg.s, tau=cfg.tau, seed=0) if mode == "lvs" else {}
    M = S.DeviceMatrix.from_host(A)
    W, H = cu(H0), cu(H0)
    out = S.iterate(M, W, H, alpha, 5, mode=mode, rule="bpp", **kw)
    _, Hr, tr = O.iterate(A, H0, H0, alpha, 5, mode, rule="bpp", **kw)
    if mode == "lvs":
        for g, o in zip(out["halves"], tr):
            assert (g["s_D"], g["s_R"], g["n_uniq"]) == (o["s_D"], o["s_R"], o["n_uniq"])
    rg, ro = O.residual(A, H.cpu().numpy()), O.residual(A, Hr)
    assert abs(rg - ro) <= 1e-4 * ro


def test_solver_lai_bpp_k64_vs_oracle():
    """LAI-BPP (the LAI variant of the paper's BPP runs) at k = 64, the c5 rank: a c5-shaped
    Gaussian-kernel problem at n = 3,000 (l = 74, q = 2), 3 LAI iterations with the exact per-row
    NLS update (k = 64: two variables per lane) vs the oracle's iterate(rule="bpp") on the GPU's
    U, Lambda: residual against the full A within 1e-4 relative."""
    d = make_input("c5", n_override=3_000)
    A, H0, alpha, cfg = d["A"], d["H0"], d["alpha"], d["cfg"]
    M = S.DeviceMatrix.from_host(A)
    U, lam = S.rangefinder(M, cfg.l, cfg.q, cfg.seed, precision="3xtf32")
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="lai", precision="3xtf32", max_iters=3, U=U, lam=lam, rule="bpp")
    sv.run(3)
    assert sv.stats()["status"] == 0
    sv.close()
    Ug, lg = U.cpu().numpy().astype(np.float64), lam.cpu().numpy()
    _, Hr, _ = O.iterate(A, H0, H0, alpha, 3, "lai", U=Ug, lam=lg, rule="bpp")
    rg, ro = O.residual(A, H.cpu().numpy()), O.residual(A, Hr)
    assert abs(rg - ro) <= 1e-4 * ro, (rg, ro)


def _drop_vertices(A, frac, tail, seed=3):
    """A with every entry of a random `frac` of the vertices and of the last `tail` vertices
    removed (rows and columns): isolated vertices, i.e. empty CSR rows, incl. an empty tail."""
    from synth.configs import CsrMatrix
    rng = np.random.default_rng(seed)
    drop = rng.random(A.n) < frac
    drop[A.n - tail:] = True
    rows = np.repeat(np.arange(A.n), np.diff(A.rowptr))
    keep = ~drop[rows] & ~drop[A.colidx]
    rowptr = np.zeros(A.n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=A.n), out=rowptr[1:])
    return CsrMatrix(A.n, rowptr, A.colidx[keep].copy(), A.val[keep].copy())


@pytest.mark.parametrize("tile", ["nnz", "rows"])
def test_csr_empty_rows(tile, monkeypatch):
    """Isolated vertices (empty CSR rows, 10% random + an empty 300-row tail): the product, the
    sampled product over all rows, one EXACT solver iteration (nnz-balanced and row SpMM), and one
    LvS half of the solver."""
    monkeypatch.setenv("SYMNMF_CSR_SPMM", tile)
    monkeypatch.setenv("SYMNMF_SWEEP", "stream")
    A0, H0, alpha = _csr_case("c2", 20_000, 16)
    A = _drop_vertices(A0, 0.1, 300)
    assert (np.diff(A.rowptr) == 0).sum() >= 2000
    M = S.DeviceMatrix.from_host(A)
    Y = S.ah(M, cu(H0)).cpu().numpy()
    assert rel(Y, O.ah(A, H0)) < 1e-5
    assert not Y[-300:].any()
    W, H = cu(H0), cu(H0)
    sv = S.Solver(M, W, H, alpha, mode="exact", max_iters=1)
    sv.run(1)
    assert sv.stats()["status"] == 0
    sv.close()
    Wr, Hr, _ = O.iterate(A, H0, H0, alpha, 1, "exact")
    assert rel(W.cpu().numpy(), Wr) < 1e-5
    assert rel(H.cpu().numpy(), Hr) < 1e-5
    # LvS: W-half vs the oracle fed the plan the GPU draws
    s_, tau = 800, 1.0 / 800
    ph = S.hybrid_sample(S.leverage_scores(cu(H0)), 16, s_, tau, 5, 0, 0).to_host()
    Gs, Ys = O.sampled_products(A, H0, ph["uniq_idx"], ph["uniq_w"])
    for path in ("stream", "fused"):
        monkeypatch.setenv("SYMNMF_SWEEP", path)
        W, H = cu(H0), cu(H0)
        sv = S.Solver(M, W, H, alpha, mode="lvs", s=s_, tau=tau, seed=5, max_iters=1)
        sv.run(1)
        assert sv.stats()["status"] == 0
        sv.close()
        assert rel(W.cpu().numpy(), O.hals_sweep(Gs, Ys, H0, H0, alpha)) < 1e-5, path


def test_csr_zero_matrix():
    """A = 0 (nnz = 0, no colidx / val storage): A F = 0 exactly, and one EXACT and one LvS solver
    iteration reduce to the regularisation pull W <- max(0, (alpha F - X G + ...)) of Eq. 2.6."""
    from synth.configs import CsrMatrix
    n, k, alpha = 3_000, 8, 0.5
    A = CsrMatrix(n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0, dtype=np.float32))
    H0 = np.random.default_rng(1).random((n, k)).astype(np.float32)
    M = S.DeviceMatrix.from_host(A)
    Y = S.ah(M, cu(H0)).cpu().numpy()
    assert not Y.any()
    lvs = dict(s=300, tau=1.0 / 300, seed=2)
    for mode, kw, spmm in (("exact", {}, "nnz"), ("exact", {}, "rows"), ("lvs", lvs, "stream"),
                           ("lvs", lvs, "fused")):
        os.environ["SYMNMF_CSR_SPMM"] = spmm
        os.environ["SYMNMF_SWEEP"] = spmm
        W, H = cu(H0), cu(H0)
        sv = S.Solver(M, W, H, alpha, mode=mode, max_iters=1, **kw)
        sv.run(1)
        assert sv.stats()["status"] == 0
        sv.close()
        Wg = W.cpu().numpy()
        if mode == "exact":
            Wr, Hr, _ = O.iterate(A, H0, H0, alpha, 1, "exact")
            assert rel(Wg, Wr) < 1e-5 and rel(H.cpu().numpy(), Hr) < 1e-5
        assert np.isfinite(Wg).all() and (Wg >= 0).all()
    os.environ.pop("SYMNMF_CSR_SPMM"); os.environ.pop("SYMNMF_SWEEP")
