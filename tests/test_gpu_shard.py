"""NEXT-4 row sharding as P logical shards on one device (paper_2402_08134_b200/shard.py):
the shards' plan pieces concatenate to the 1-shard plan bit for bit given the same scores, and
sharded EXACT / LvS iterations match the unsharded computation.  Unmeasured on multi-GPU hardware
(gpurun has one GPU); the collective plumbing for one shard per rank is DistComm (NCCL / gloo)."""
import numpy as np
import pytest

import oracle as O
from synth import make_input
from synth.configs import init_factor, mean_entry

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2402_08134_b200 import symnmf as S  # noqa: E402
from paper_2402_08134_b200 import shard as SH  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def cu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("n,k,s,P", [(100_000, 16, 2000, 2), (100_000, 16, 2000, 4), (2_000_000, 32, 20_000, 3),
                                     (2_000_000, 32, 20_000, 4), (5_003, 8, 300, 4)])
def test_shard_plans_concatenate_to_the_global_plan(n, k, s, P):
    """P:711-741 / readings Z1-Z6: per-shard masses, their exclusive scan (exact uint64), and each
    shard's plan part from the global draws -> concatenation == symnmf_hybrid_sample, bit for bit."""
    F = (np.random.default_rng(n + P).random((n, k)) ** 3).astype(np.float32)
    lev = S.leverage_scores(cu(F))
    g = S.hybrid_sample(lev, k, s, 1.0 / s, 7, 3, 1).to_host()
    blocks = SH.row_blocks(n, P)
    sums = [S.hybrid_shard_sums(lev[r0:r1], k, 1.0 / s) for r0, r1 in blocks]
    offs, W, sD = SH.mass_offsets(sums)
    assert W == g["W"] and sD == g["s_D"]
    U, Wt = [], []
    for (r0, r1), off in zip(blocks, offs):
        pl = S.hybrid_shard_plan(lev[r0:r1], r0, k, s, 1.0 / s, 7, 3, 1, off, W, sD).to_host()
        assert pl["s_R"] == g["s_R"]
        U.append(pl["uniq_idx"]); Wt.append(pl["uniq_w"])
    assert np.array_equal(np.concatenate(U), g["uniq_idx"])
    assert np.array_equal(np.concatenate(Wt), g["uniq_w"])


def _case(cfgname, n, k, seed=5):
    d = make_input(cfgname, n_override=n)
    A = d["A"]
    H0 = init_factor(n, k, mean_entry(A), np.random.default_rng(seed))
    return A, H0, d["alpha"]


@pytest.mark.parametrize("cfgname,n,k,P", [("c2", 100_000, 16, 2), ("c2", 100_000, 16, 4), ("c4", 200_000, 32, 2),
                                           ("c4", 200_000, 32, 4)])
def test_sharded_exact_iteration_matches_oracle(cfgname, n, k, P):
    """EXACT: allgather F, block rows of A F, allreduced Gram, block sweeps.  Two iterations,
    each half vs the oracle's fp64 half fed the GPU's own previous factors (1e-5 relative): the
    per-half protocol isolates the sharded arithmetic from the fp32 amplification of earlier halves
    (at c4 n = 200k the unsharded solver's H after one whole iteration is itself 1.2e-5 from the
    oracle's -- DESIGN.md sec. 5)."""
    A, H0, alpha = _case(cfgname, n, k)
    A64 = O.as_f64(A)
    sv = SH.ShardedSolver(A, H0, alpha, SH.LocalComm(P), mode="exact")
    for it in range(2):
        for side in (0, 1):
            W0, H0_ = (t.cpu().numpy().astype(np.float64) for t in sv.factors())
            sv.half(it, side)
            W, H = (t.cpu().numpy() for t in sv.factors())
            Wr, Hr, _ = O.half_step(A64, W0, H0_, alpha, it, side, "exact")
            got, ref = (W, Wr) if side == 0 else (H, Hr)
            assert rel(got, ref) < 1e-5, (it, side, rel(got, ref))


@pytest.mark.parametrize("cfgname,n,k,s,P", [("c2", 100_000, 16, 2000, 2), ("c2", 100_000, 16, 2000, 4),
                                             ("c4", 200_000, 32, 2000, 2), ("c4", 200_000, 32, 2000, 4)])
def test_sharded_lvs_half_matches_oracle_and_global_plan(cfgname, n, k, s, P):
    """LvS: the sharded half's plan equals symnmf_hybrid_sample on its own (gathered) scores
    bit for bit, its scores match the unsharded ones (Z21, 1e-5), and the updated factor equals the
    oracle's sampled products + sweep fed that plan (1e-5)."""
    A, H0, alpha = _case(cfgname, n, k)
    tau = 1.0 / s
    sv = SH.ShardedSolver(A, H0, alpha, SH.LocalComm(P), mode="lvs", s=s, tau=tau, seed=3)
    sv.half(0, 0)
    last = sv.last
    lev = last["lev"]
    assert rel(lev.cpu().numpy(), S.leverage_scores(cu(H0)).cpu().numpy()) < 1e-5
    g = S.hybrid_sample(lev, k, s, tau, 3, 0, 0).to_host()
    assert np.array_equal(last["uniq_idx"].cpu().numpy(), g["uniq_idx"])
    assert np.array_equal(last["uniq_w"].cpu().numpy(), g["uniq_w"])
    assert last["s_D"] == g["s_D"] and last["W"] == g["W"]
    W, _ = sv.factors()
    Gs, Ys = O.sampled_products(A, H0, g["uniq_idx"], g["uniq_w"])
    assert rel(W.cpu().numpy(), O.hals_sweep(Gs, Ys, H0, H0, alpha)) < 1e-5


@pytest.mark.parametrize("n,l,k,P", [(5_003, 20, 16, 1), (5_003, 20, 16, 3), (40_000, 74, 64, 2), (40_000, 74, 64, 4)])
def test_sharded_lai_blocks_and_iteration_match_oracle(n, l, k, P):
    """LAI on row blocks (Eq. 3.1): sum_b U_b^T F_b then U_b (Lambda Z) equals the oracle's
    U (Lambda (U^T F)) (1e-5), with one block it equals symnmf_lai_ah, and two sharded iterations match
    the oracle's fp64 LAI halves fed the GPU's own previous factors (per-half protocol, 1e-5)."""
    r = np.random.default_rng(n + l + P)
    U = np.linalg.qr(r.standard_normal((n, l)))[0].astype(np.float32)
    lam = np.sort(r.random(l) * 50)[::-1].copy()
    lam[-3:] *= -0.1                                   # Apx-EVD eigenvalues may be negative
    H0 = init_factor(n, k, 0.5, np.random.default_rng(5))
    Ud, lamd = cu(U), cu(lam)
    blocks = SH.row_blocks(n, P)
    Hd = cu(H0)
    Z = sum(S.lai_project_rows(Ud[r0:r1], Hd[r0:r1]) for r0, r1 in blocks)
    assert rel(Z.cpu().numpy(), U.astype(np.float64).T @ H0.astype(np.float64)) < 1e-6
    Y = torch.cat([S.lai_apply_rows(Ud[r0:r1], lamd, Z) for r0, r1 in blocks]).cpu().numpy()
    assert rel(Y, O.lai_apply(U, lam, H0)) < 1e-5
    if P == 1:
        assert np.array_equal(Y, S.lai_ah(Ud, lamd, Hd).cpu().numpy())
    alpha = 1.0                                        # any alpha >= 0 (the paper takes max(A))
    sv = SH.ShardedSolver(None, H0, alpha, SH.LocalComm(P), mode="lai", lai=(U, lam))
    for it in range(2):
        for side in (0, 1):
            W0, H0_ = (t.cpu().numpy().astype(np.float64) for t in sv.factors())
            sv.half(it, side)
            W, H = (t.cpu().numpy() for t in sv.factors())
            Wr, Hr, _ = O.half_step(None, W0, H0_, alpha, it, side, "lai", U=U, lam=lam)
            got, ref = (W, Wr) if side == 0 else (H, Hr)
            assert rel(got, ref) < 1e-5, (it, side, rel(got, ref))
