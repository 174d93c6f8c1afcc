"""World-size-2 gloo tests of the multi-process host logic (CPU only).

1. bench.py's replica protocol: barrier, device time max-reduced over ranks,
   value = ranks * steps / max time (replicas only).
2. The row-sharded hybrid sampler of the NEXT-4 design: each rank
   owns a contiguous row block of the score vector, builds its integer masses
   and inclusive prefix locally, the block totals are all-gathered into
   exclusive offsets, every rank evaluates all s_R Philox draws and resolves
   those whose target falls into its prefix range.  Integer prefix sums are
   associative, so the gathered plan must be bit-identical to the
   single-process plan (oracle.build_plan).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, ws, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)


def _replica_worker(rank, ws, port, q):
    import bench
    _init(rank, ws, port)
    t_ms = 10.0 + 5.0 * rank            # per-rank device time of K steps
    dist.barrier()
    t = bench.max_over_ranks(dist, t_ms, torch.device("cpu"))
    steps = 100
    q.put((rank, t, ws * steps / (t / 1e3)))
    dist.destroy_process_group()


def test_replica_timing_is_max_over_ranks():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_replica_worker, args=(ws, port, q), nprocs=ws, join=True)
    out = sorted(q.get() for _ in range(ws))
    assert all(o[1] == 15.0 for o in out)                       # max over ranks
    assert all(abs(o[2] - 2 * 100 / 0.015) < 1e-6 for o in out)


def _sharded_plan_worker(rank, ws, port, lev, k, s, tau, seed, it, side, q):
    _init(rank, ws, port)
    n = lev.size
    lo, hi = rank * n // ws, (rank + 1) * n // ws
    l = lev[lo:hi].astype(np.float64)
    T = tau * k
    det = l >= T
    w = np.floor(l * 2.0 ** 40).astype(np.uint64)
    w[det] = 0
    P_local = np.cumsum(w, dtype=np.uint64)
    tot = torch.tensor([int(P_local[-1]) if P_local.size else 0, int(det.sum())], dtype=torch.int64)
    allt = [torch.zeros(2, dtype=torch.int64) for _ in range(ws)]
    dist.all_gather(allt, tot)
    masses = [int(t[0]) for t in allt]
    sDs = [int(t[1]) for t in allt]
    off = sum(masses[:rank])
    W = sum(masses)
    s_D = sum(sDs)
    s_R = max(0, s - s_D) if W > 0 else 0
    j = np.arange(s_R, dtype=np.uint64)
    u, _ = O.philox_u64(j, 2 * it + side, 0, seed)              # every rank draws all s_R targets
    t = O.mulhi64(u, W) if s_R else np.empty(0, np.uint64)
    mine = (t >= np.uint64(off)) & (t < np.uint64(off + masses[rank]))
    local_idx = np.searchsorted(P_local, t[mine] - np.uint64(off), side="right") + lo
    q.put((rank, np.nonzero(det)[0] + lo, np.nonzero(mine)[0], local_idx, W, s_D, s_R))
    dist.destroy_process_group()


@pytest.mark.parametrize("n,k,s,tau", [(5000, 8, 300, 1 / 300), (4099, 4, 200, 1.0)])
def test_row_sharded_plan_equals_single_process_plan(n, k, s, tau):
    rng = np.random.default_rng(n)
    F = rng.random((n, k)) ** 4
    lev = O.leverage_scores(F).astype(np.float32)
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_sharded_plan_worker, args=(ws, port, lev, k, s, tau, 7, 3, 1, q), nprocs=ws, join=True)
    parts = sorted(q.get() for _ in range(ws))
    ref = O.build_plan(lev, k, s, tau, 7, 3, 1)
    det = np.concatenate([p[1] for p in parts])
    assert np.array_equal(det, ref["det_idx"])
    s_R = parts[0][6]
    draws = np.empty(s_R, dtype=np.int64)
    for p in parts:
        draws[p[2]] = p[3]
    assert parts[0][4] == ref["W"] and parts[0][5] == ref["s_D"] and s_R == ref["s_R"]
    assert np.array_equal(draws, ref["draw_idx"])


def _distcomm_worker(rank, ws, port, q):
    from paper_2402_08134_b200.shard import DistComm, mass_offsets
    _init(rank, ws, port)
    c = DistComm()
    # variable-length concatenation (plan rows of different sizes per shard), in rank order
    x = torch.arange(3 + 2 * rank, dtype=torch.int32) + 100 * rank
    cat = c.allgather_cat([x])[0]
    # k x k Gram partials: fp64 sum
    g = c.allreduce_sum([torch.full((2, 2), 1.5 * (rank + 1), dtype=torch.float64)])[0]
    # the shards' exact integer masses (uint64 range), s_D and theta, and their exclusive scan
    sums = c.allgather_obj([((1 << 62) + 7 * rank, 3 + rank, 0.25 * rank)])[0]
    offs, W, sD = mass_offsets(sums)
    q.put((rank, cat.tolist(), g.tolist(), offs, W, sD))
    dist.destroy_process_group()


def test_shard_distcomm_collectives_over_gloo():
    """paper_2402_08134_b200.shard.DistComm (one shard per rank) over gloo, world size 2: the
    variable-length all-gather the shards' plan rows go through, the Gram allreduce, and the exact
    uint64 exclusive scan of the shards' masses."""
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_distcomm_worker, args=(ws, port, q), nprocs=ws, join=True)
    out = sorted(q.get() for _ in range(ws))
    for rank, cat, g, offs, W, sD in out:
        assert cat == [0, 1, 2, 100, 101, 102, 103, 104]
        assert g == [[4.5, 4.5], [4.5, 4.5]]
        assert offs == [0, (1 << 62)] and W == (1 << 63) + 7 and sD == 7
