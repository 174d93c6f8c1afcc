"""NEXT-4: row-sharded LvS / EXACT iterations over the C ABI's shard building blocks.

A shard owns a contiguous row block [r0, r1) of A (CSR rows with global column indices), W and H.
One half-iteration (Alg. LvS-SymNMF; P:181 for EXACT):

    LvS    G_b = F_b^T F_b  --allreduce-->  G ;  l_b = scores(F_b; G)
           (W_b, s_D,b, theta_b) --allgather--> exclusive scan of the integer masses W_b gives each
           shard its offset inside the global prefix; its part of the plan (global draws landing in
           its mass range, weights with the global W, s_R)
           (Z_b, G_s,b) for its plan rows --allgather / allreduce--> (U, Z), G_s
           Y_s rows of the block as a pull over its CSR rows (no exchange of A)
           X_b <- sweep(G_s, Y_s,b, F_b, X_b)
    EXACT  F --allgather--> F_all;  Y_b = A_b F_all;  G = allreduce(G_b);  X_b <- sweep(G, Y_b, F_b, X_b)
    LAI    Z_b = U_b^T F_b (l x k) --allreduce--> Z;  Y_b = U_b (Lambda Z);  G = allreduce(G_b);
           X_b <- sweep(G, Y_b, F_b, X_b)                                          (Eq. 3.1)

The collectives are plumbing: `LocalComm` holds P logical shards in one process (one device; sums in
shard order, concatenation), `DistComm` one shard per rank over torch.distributed (NCCL for CUDA
tensors, gloo on CPU).  Every arithmetic step runs in libsymnmf's kernels; integer masses and offsets
are exact, so the concatenated plan equals the 1-shard plan given the same scores.
"""
from __future__ import annotations

import numpy as np
import torch

from . import symnmf as S


def row_blocks(n: int, P: int):
    """Contiguous row blocks [r_p, r_{p+1}) with r_p = floor(n p / P)."""
    return [(n * p // P, n * (p + 1) // P) for p in range(P)]


def mass_offsets(sums):
    """Exclusive prefix of the shards' uint64 masses, their total, and the global s_D (exact ints)."""
    offs, run = [], 0
    for w, _, _ in sums:
        offs.append(run)
        run += int(w)
    return offs, run, sum(int(sd) for _, sd, _ in sums)


class LocalComm:
    """P logical shards in one process: the collectives are shard-ordered sums and concatenations."""

    def __init__(self, P: int):
        self.P = P
        self.shards = list(range(P))

    def allreduce_sum(self, parts):
        tot = parts[0].clone()
        for x in parts[1:]:
            tot += x
        return [tot] * len(parts)

    def allgather_cat(self, parts):
        cat = torch.cat(list(parts))
        return [cat] * len(parts)

    def allgather_obj(self, objs):
        return [list(objs)] * len(objs)


class DistComm:
    """One shard per rank of the default torch.distributed group (NCCL over NVLink for CUDA tensors)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.P = dist.get_world_size()
        self.shards = [dist.get_rank()]

    def allreduce_sum(self, parts):
        t = parts[0].clone()
        self.dist.all_reduce(t)
        return [t]

    def allgather_cat(self, parts):
        x = parts[0].contiguous()
        n = torch.tensor([x.shape[0]], dtype=torch.int64, device=x.device)
        sizes = [torch.zeros_like(n) for _ in range(self.P)]
        self.dist.all_gather(sizes, n)
        sizes = [int(v.item()) for v in sizes]
        m = max(sizes + [1])
        pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        pad[:x.shape[0]] = x
        bufs = [torch.empty_like(pad) for _ in range(self.P)]
        self.dist.all_gather(bufs, pad)
        return [torch.cat([b[:c] for b, c in zip(bufs, sizes)])]

    def allgather_obj(self, objs):
        out = [None] * self.P
        self.dist.all_gather_object(out, objs[0])
        return [out]


class ShardedSolver:
    """Row-sharded EXACT / LvS iterations on CSR A, or LAI iterations on (U, lambda) (the shards this
    process owns, per `comm`).

    A: synth.CsrMatrix (host; each shard takes its rows), H0 (host n x k fp32), W0 = H0.
    mode="lai": A is None and lai=(U, lam) holds the range finder's factors (host or device, n x l
    fp32 and l fp64; each shard takes its rows of U)."""

    def __init__(self, A, H0, alpha: float, comm, mode="lvs", s=0, tau=1.0, seed=0, device="cuda", lai=None):
        self.comm, self.mode, self.alpha = comm, mode, float(alpha)
        self.s, self.tau, self.seed = int(s), float(tau), int(seed)
        self.n, self.k = H0.shape[0], H0.shape[1]
        self.blocks = row_blocks(self.n, comm.P)
        self.M, self.W, self.H, self.U = [], [], [], []
        if mode == "lai":
            U, lam = (torch.as_tensor(x) for x in lai)
            self.lam = lam.to(device=device, dtype=torch.float64).contiguous()
        for p in comm.shards:
            r0, r1 = self.blocks[p]
            if mode == "lai":
                self.U.append(U[r0:r1].to(device=device, dtype=torch.float32).contiguous())
                self.W.append(torch.from_numpy(np.ascontiguousarray(H0[r0:r1])).to(device))
                self.H.append(torch.from_numpy(np.ascontiguousarray(H0[r0:r1])).to(device))
                continue
            e0, e1 = int(A.rowptr[r0]), int(A.rowptr[r1])
            rp = torch.from_numpy((A.rowptr[r0:r1 + 1] - e0).astype(np.int64)).to(device)
            ci = torch.from_numpy(np.ascontiguousarray(A.colidx[e0:e1])).to(device)
            va = torch.from_numpy(np.ascontiguousarray(A.val[e0:e1])).to(device)
            self.M.append(S.DeviceMatrix(rowptr=rp, colidx=ci, val=va, n=r1 - r0))
            self.W.append(torch.from_numpy(np.ascontiguousarray(H0[r0:r1])).to(device))
            self.H.append(torch.from_numpy(np.ascontiguousarray(H0[r0:r1])).to(device))
        self.last = None   # the last half's global plan and the shards' scores (tests)

    def half(self, it: int, side: int):
        c = self.comm
        F = self.H if side == 0 else self.W
        X = self.W if side == 0 else self.H
        G = c.allreduce_sum([S.gram(f) for f in F])
        if self.mode == "lai":   # Y_b = U_b (Lambda sum_b U_b^T F_b): one l x k allreduce (Eq. 3.1)
            Z = c.allreduce_sum([S.lai_project_rows(u, f) for u, f in zip(self.U, F)])
            for i in range(len(F)):
                Y = S.lai_apply_rows(self.U[i], self.lam, Z[i])
                S.hals_sweep(G[i], Y, F[i], X[i], self.alpha)
            return
        if self.mode == "exact":
            F_all = c.allgather_cat(F)
            for i in range(len(F)):
                Y = torch.empty_like(F[i])
                S.ah(self.M[i], F_all[i], out=Y)     # block rows, global columns of F_all
                S.hals_sweep(G[i], Y, F[i], X[i], self.alpha)
            return
        levs = [S.leverage_scores_gram(f, g) for f, g in zip(F, G)]
        sums = c.allgather_obj([S.hybrid_shard_sums(l, self.k, self.tau) for l in levs])
        plans, Zs, Gss = [], [], []
        for i, p in enumerate(c.shards):
            offs, W_tot, sD_tot = mass_offsets(sums[i])
            r0 = self.blocks[p][0]
            pl = S.hybrid_shard_plan(levs[i], r0, self.k, self.s, self.tau, self.seed, it, side, offs[p], W_tot,
                                     sD_tot)
            nu = int(pl.counts[2].item())
            Z, Gs = S.plan_rows_scaled(F[i], r0, pl)
            plans.append(pl)
            Zs.append(Z[:nu])
            Gss.append(Gs)
        Gs = c.allreduce_sum(Gss)
        U = c.allgather_cat([pl.uniq_idx[:int(pl.counts[2].item())] for pl in plans])
        Wt = c.allgather_cat([pl.uniq_w[:int(pl.counts[2].item())] for pl in plans])
        Z = c.allgather_cat(Zs)
        for i in range(len(F)):
            Y = S.sampled_ah_rows(self.M[i], self.n, U[i], Z[i], self.k)
            S.hals_sweep(Gs[i], Y, F[i], X[i], self.alpha)
        self.last = {"uniq_idx": U[0], "uniq_w": Wt[0], "lev": c.allgather_cat(levs)[0],
                     "s_D": sum(int(x[1]) for x in sums[0]), "W": mass_offsets(sums[0])[1]}

    def run(self, iters: int, first_iter: int = 0):
        for t in range(iters):
            self.half(first_iter + t, 0)
            self.half(first_iter + t, 1)

    def factors(self):
        """(W, H) of the whole problem (gathered)."""
        return self.comm.allgather_cat(self.W)[0], self.comm.allgather_cat(self.H)[0]
