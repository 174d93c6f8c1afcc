#!/usr/bin/env python
"""Benchmark of the randomized-SymNMF hot path on B200 (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--mode lvs|exact|lai]
                [--impl ours|reference]

A step is one full iteration (W-half + H-half) of the solver of config
`--config` (default c4 -- the largest single-GPU configuration of BASELINE.json with both modes of the
metric -- mode LvS: CholeskyQR scores, hybrid plan, sampled Gram, sampled product, HALS sweep with
the next Gram fused), replayed
from the solver's captured CUDA graph with inputs resident in HBM.  L2 is
flushed (256 MiB write) before every timed step.  N > 1 runs N independent
replicas (the single-GPU north star does not shard; weak
scaling, no collective on the data path), timed on the device as the max over
ranks.  Only tests/, smoke() and this file's cpu_baseline / reference legs
import oracle/.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SymNMF iters/sec (exact & LvS); A·H / sampled SpMM HBM GB/s vs B200 peak"
UNIT = "iters/s"
SLEEP_CYCLES = 400_000   # ~0.2 ms: keeps the GPU busy while the host enqueues, so events time the device
TF32_OVER_BF16 = 0.5     # nominal dense tf32 / bf16 ratio (B200_PROFILING.md: 1.1 vs 2.25 PFLOP/s)
ALU_BOUND = {"lai_fused"}   # kernels whose roofline is fp32 SIMT arithmetic
# Measured ceiling of global float reductions into random 128-byte rows of an L2-resident range on this
# pool's B200 (tools/red_bench.cu, profiles/r2_red_bench.txt: 49.2 G rows/s = 6.3 TB/s of atomic payload,
# the same for red.v4 and red.v2, 1965 MHz): what bounds the sampled CSR scatter, whose DRAM is ~20% busy.
L2_ATOMIC_ROWS_PER_S = 49.2e9
# Same tool, "ld" lines: 1e8 gathers of random 128-byte rows run at 75 G rows/s (9.6 TB/s) from an L2-resident
# range and 66.5 G rows/s (8.5 TB/s) from a 256 MB one -- the L2 slices' throughput, not HBM, caps the exact
# CSR product's F gathers at k = 32 (one 128 B row of F per nonzero).
L2_GATHER_ROWS_PER_S = 66.5e9


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--mode", default=None, choices=[None, "lvs", "exact", "lai"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rule", default="hals", choices=["hals", "bpp"], help="Update(): HALS sweep or BPP (NEXT-1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--profile-only", action="store_true", help="warmup + timed loop only (for ncu)")
    a = ap.parse_args()
    if a.mode is None:
        a.mode = "lai" if a.config == "c5" else "lvs"
    return a


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        rows = self.rows
        load = [r for r in rows if (num(r[2]) or 0) > 0] or rows
        sm = [num(r[0]) for r in load if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if num(r[1]) is not None]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(load)}


# ------------------------------------------------------------------ distributed plumbing
def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if ws > 1:
        import torch.distributed as dist
        if args.impl == "ours":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
        pg = dist
    return ws, rank, local, pg


def max_over_ranks(pg, value, dev):
    if not pg:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ algorithmic bytes per launch
def kernel_cost(name, n, k, nnz=0, nnz_u=0, n_u=0, l=0, zeroY=False):
    """(algorithmic bytes, flops) one launch must move / compute (SURVEY §8(d) per-unit figures)."""
    if name == "spmm_csr":
        return 8 * nnz + 8 * (n + 1) + 8 * n * k, 2 * nnz * k
    if name in ("gemm_3xtf32", "gemm_fp32"):
        return 4 * n * n + 8 * n * k, 2 * n * n * k
    if name == "sampled_ah_csr":
        return 8 * nnz_u + 16 * n_u + 4 * n_u * k + 4 * n * k, 2 * nnz_u * k
    if name == "sampled_ah_dense":
        return 4 * n_u * n + 4 * n_u * k + 4 * n * k, 2 * n * n_u * k
    if name == "csr_tile_exact":   # spmm + sweep fused: Y never leaves the SM, F counted once
        return 8 * nnz + 8 * (n + 1) + 12 * n * k, 2 * nnz * k + 2 * n * k * k
    if name == "csr_tile_lvs":     # sampled product (SURVEY §8(d) N8 bytes) + sweep, fused
        return 8 * nnz_u + 16 * n_u + 4 * n_u * k + 12 * n * k, 2 * nnz_u * k + 2 * n * k * k
    if name == "bpp_update":   # read Y, F, write X (+ Y re-zero in LvS); pivoting solves are fp64 ALU work
        return (20 if zeroY else 16) * n * k, None
    if name == "hals_sweep":   # read Y, X, F, write X (a re-zero of Y is not method bytes)
        return 16 * n * k, 2 * n * k * k
    if name == "leverage":
        return 4 * n * k + 4 * n, n * k * k
    if name == "sampled_gram":
        return n_u * (4 * k + 12), n_u * k * k
    if name == "samp_prefix":
        return 4 * n + 8 * n, 0
    if name == "samp_draws":
        return None, None
    if name in ("samp_uniq_count", "samp_uniq_write"):
        return 8 * n, 0
    if name == "lai_fused":   # U tile, F tile, X read + write; flops: U M, sweep, X^T X, U^T X
        return 4 * n * l + 12 * n * k, 2 * n * (2 * l * k + k * k + k * (k + 1) // 2)
    if name == "lai_utf":
        return 4 * n * l + 4 * n * k, 2 * n * l * k
    if name == "lai_uz":
        return 4 * n * l + 4 * n * k, 2 * n * l * k
    return None, None


# ------------------------------------------------------------------ workload description (both arms)
def precision_of(d):
    A = d["A"]
    dense = not hasattr(A, "rowptr")
    return "3xtf32" if dense and d["n"] % 4 == 0 else "fp32"


def config_dict(args, d, ws):
    """The `config` object of the JSON line; identical in our arm and the reference arm."""
    cfg, A, n = d["cfg"], d["A"], d["n"]
    dense = not hasattr(A, "rowptr")
    lvs = args.mode == "lvs"
    return {"workload": args.config, "n": n, "nnz": int(n * n if dense else A.nnz), "k": cfg.k, "mode": args.mode,
            "rule": args.rule, "precision": precision_of(d), "s": cfg.s if lvs else None,
            "tau": cfg.tau if lvs else None, "l": cfg.l or None, "q": cfg.q or None,
            "l2": "flushed (256 MiB write) before every timed step", "parallelism": f"replicas{ws}",
            "graph": "per-iteration CUDA graph replay (PDL edges only below 2^15 rows)"}


# ------------------------------------------------------------------ reference arm: the oracle on host cores
class OracleRun:
    """The fp64 oracle (oracle/) advanced one half-iteration at a time (oracle.half_step, the body of
    oracle.iterate), so that a bounded sample of the workload can be timed."""

    def __init__(self, args, d):
        import numpy as np
        import oracle as O
        self.O, self.args, self.d = O, args, d
        cfg = d["cfg"]
        self.kw = {}
        if args.mode == "lvs":
            self.kw = dict(s=cfg.s, tau=cfg.tau, seed=cfg.seed)
        elif args.mode == "lai":
            U, lam, _ = O.rangefinder(d["A"], cfg.l, cfg.q, seed=cfg.seed)
            self.kw = dict(U=U, lam=lam)
        self.A64 = O.as_f64(d["A"]) if args.mode != "lai" else None
        self.W = d["H0"].astype(np.float64)
        self.H = d["H0"].astype(np.float64)
        self.halves = 0

    def half(self):
        it, side = divmod(self.halves, 2)
        self.W, self.H, _ = self.O.half_step(self.A64, self.W, self.H, self.d["alpha"], it, side, self.args.mode,
                                             rule=self.args.rule, **self.kw)
        self.halves += 1


def run_reference(args, rank, ws):
    """The oracle as it stands, on this host's cores: one step = one half-iteration (W- or H-update,
    alternating), so value = steps / 2 / seconds iterations per second."""
    from synth import make_input
    if rank != 0:
        return None
    d = make_input(args.config)
    run = OracleRun(args, d)
    for _ in range(args.warmup):
        run.half()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run.half()
    dt = time.perf_counter() - t0
    v = args.steps / 2 / dt
    sample = (f"{args.steps} oracle half-iterations (after {args.warmup} untimed) of {args.config} {args.mode} "
              f"at full n; one step = one half-iteration")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, d, ws),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def cpu_baseline(args, d):
    """The oracle on a bounded sample: as many half-iterations of the full workload as fit in
    --cpu-budget seconds (at least one)."""
    run = OracleRun(args, d)
    t0 = time.perf_counter()
    while True:
        run.half()
        if time.perf_counter() - t0 > args.cpu_budget:
            break
    dt = time.perf_counter() - t0
    return {"value": run.halves / 2 / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"first {run.halves} oracle half-iterations of {args.config} {args.mode} (full n), "
                      f"~{args.cpu_budget:.0f} s budget"}


# ------------------------------------------------------------------ our arm
def run_ours(args, ws, rank, local, pg):
    import numpy as np
    import torch
    from paper_2402_08134_b200 import symnmf as S
    from synth import make_input

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    d = make_input(args.config)
    cfg = d["cfg"]
    A, H0, alpha = d["A"], d["H0"], d["alpha"]
    n, k = d["n"], cfg.k
    dense = not hasattr(A, "rowptr")
    precision = precision_of(d)
    M = S.DeviceMatrix.from_host(A)
    W = torch.from_numpy(H0).to(dev)
    H = torch.from_numpy(H0).to(dev)
    kw = {}
    extra = {}
    if args.mode == "lvs":
        kw = dict(s=cfg.s, tau=cfg.tau, seed=cfg.seed)
    elif args.mode == "lai":
        # the range finder (Alg. RRF + Apx-EVD) runs once per solve: first call (module load,
        # descriptor setup) and a warm call are both reported
        for key in ("rangefinder_first_ms", "rangefinder_ms"):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            U, lam = S.rangefinder(M, cfg.l, cfg.q, cfg.seed, precision=precision)
            e1.record()
            torch.cuda.synchronize()
            extra[key] = e0.elapsed_time(e1)
        kw = dict(U=U, lam=lam)
    total = args.warmup + args.steps
    solver = S.Solver(M, W, H, alpha, mode=args.mode, precision=precision, max_iters=total, rule=args.rule, **kw)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        solver.run(1)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for e0, e1 in evs:
        flush.zero_()
        torch.cuda._sleep(SLEEP_CYCLES)
        e0.record(stream)
        solver.run(1)
        e1.record(stream)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    t_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    st = solver.stats()
    if st["status"] != 0:
        raise RuntimeError(f"device status {st['status']}")
    kernels_per_iter, memsets_per_iter = solver.graph_nodes()
    if args.profile_only:
        clocks.stop()
        return None
    t_max = max_over_ranks(pg, t_ms, dev)
    value = ws * args.steps / (t_max / 1e3)

    # the other half of the metric: exact-product iterations (LvS configs) with the same protocol
    if args.mode == "lvs":
        ex_steps = max(3, min(args.steps, 30))
        W2, H2 = torch.from_numpy(H0).to(dev), torch.from_numpy(H0).to(dev)
        sx = S.Solver(M, W2, H2, alpha, mode="exact", precision=precision, max_iters=args.warmup + ex_steps,
                      rule=args.rule)
        sx.run(args.warmup)
        torch.cuda.synchronize()
        acc = 0.0
        for _ in range(ex_steps):
            flush.zero_()
            torch.cuda._sleep(SLEEP_CYCLES)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream); sx.run(1); e1.record(stream)
            e1.synchronize()
            acc += e0.elapsed_time(e1)
        extra["exact_iters_per_s"] = ws * ex_steps / (max_over_ranks(pg, acc, dev) / 1e3)
        extra["exact_precision"] = precision
        sx.close()

    # per-kernel device times of the same kernels (eager evented iterations)
    prof = solver.profile(iters=5)
    per = {}
    for name, ms in prof:
        per.setdefault(name, []).append(ms)
    share = {nm: sum(v) for nm, v in per.items()}
    iter_ms = sum(share.values())
    dom = max((nm for nm in share if nm != "bump_iter"), key=share.get)
    dom_ms = statistics.mean(per[dom])
    nnz = A.nnz if not dense else n * n
    nnz_u = n_u = 0
    if args.mode == "lvs":
        halves = st["halves"][2 * args.warmup:] or st["halves"]
        n_u = int(round(statistics.mean(h["n_uniq"] for h in halves)))
        if not dense:   # nnz of a representative plan: the final H's own plan
            lev = S.leverage_scores(H)
            ph = S.hybrid_sample(lev, k, cfg.s, cfg.tau, cfg.seed, total, 0).to_host()
            nnz_u = int(np.sum(A.rowptr[ph["uniq_idx"] + 1] - A.rowptr[ph["uniq_idx"]]))
    by, fl = kernel_cost(dom, n, k, nnz=nnz, nnz_u=nnz_u, n_u=n_u, l=cfg.l, zeroY=args.mode == "lvs")
    pk, which = peaks()
    if dom in ALU_BOUND:   # fp32 SIMT-bound: 148 SMs x 128 FMA/clk x 2 x max SM clock
        alu_peak = 148 * 128 * 2 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        roof = {"bound": "alu", "kernel": dom, "achieved": fl / (dom_ms * 1e-3) / 1e12 if fl else None,
                "peak": alu_peak, "unit": "TFLOP/s", "frac": None, "traffic": None, "algorithmic_flops": fl,
                "algorithmic_bytes": by, "kernel_ms": dom_ms, "share_of_step": share[dom] / iter_ms,
                "peak_source": "derived: 148 SMs x 128 fp32 FMA/clk x 2 x sm_max_mhz (MEASURED_PEAKS.json)"}
        if roof["achieved"]:
            roof["frac"] = roof["achieved"] / alu_peak
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": None, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": None,
                "traffic": None, "algorithmic_bytes": by, "kernel_ms": dom_ms, "share_of_step": share[dom] / iter_ms,
                "peak_source": f"{which} (MEASURED_PEAKS.json hbm_gbs: copy bandwidth)"}
        if by:
            roof["achieved"] = by / (dom_ms * 1e-3) / 1e9
            roof["frac"] = roof["achieved"] / pk["hbm_gbs"]
    if dom == "sampled_ah_csr" and nnz_u and k == 32:   # one 128 B row of atomics per sampled nonzero
        rows_s = nnz_u / (dom_ms * 1e-3)
        roof["l2_atomic"] = {"achieved": rows_s / 1e9, "peak": L2_ATOMIC_ROWS_PER_S / 1e9, "unit": "G row-adds/s",
                             "frac": rows_s / L2_ATOMIC_ROWS_PER_S,
                             "peak_source": "tools/red_bench.cu on B200 (profiles/r2_red_bench.txt)"}
    if dom == "spmm_csr" and k == 32 and 4 * n * k > (100 << 20):   # one 128 B row of F gathered per nonzero
        rows_s = nnz / (dom_ms * 1e-3)
        roof["l2_gather"] = {"achieved": rows_s / 1e9, "peak": L2_GATHER_ROWS_PER_S / 1e9, "unit": "G row-gathers/s",
                             "frac": rows_s / L2_GATHER_ROWS_PER_S,
                             "peak_source": "tools/red_bench.cu on B200 (profiles/r2_red_bench.txt, 256 MB range)"}
    if dom in ("gemm_3xtf32",) and fl:
        tf32 = pk.get("bf16_tflops", 1590.0) * TF32_OVER_BF16 / 3.0
        roof["tensor_3xtf32_tflops"] = {"achieved": fl / (dom_ms * 1e-3) / 1e12, "peak": tf32,
                                        "frac": fl / (dom_ms * 1e-3) / 1e12 / tf32}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            roof["traffic"] = json.load(open(tpath)).get(args.config, {}).get(dom)
        except Exception:
            pass
    kernels = {}
    for nm, v in per.items():
        b_, _ = kernel_cost(nm, n, k, nnz=nnz, nnz_u=nnz_u, n_u=n_u, l=cfg.l, zeroY=args.mode == "lvs")
        kernels[nm] = {"ms": round(statistics.mean(v), 5), "launches_per_step": len(v),
                       "gbs": round(b_ / (statistics.mean(v) * 1e-3) / 1e9, 1) if b_ else None}

    # end to end through the public API: pinned host inputs in, factors out, every step
    e2e = None
    if not args.no_e2e:
        if not dense:
            host_in = [torch.from_numpy(A.rowptr).pin_memory(), torch.from_numpy(A.colidx).pin_memory(),
                       torch.from_numpy(A.val).pin_memory()]
            dev_in = [M.rowptr, M.colidx, M.val]
        else:
            host_in = [torch.from_numpy(A).pin_memory()]
            dev_in = [M.dense]
        hW, hH = torch.from_numpy(H0).pin_memory(), torch.from_numpy(H0).pin_memory()
        oW, oH = torch.empty_like(hW).pin_memory(), torch.empty_like(hH).pin_memory()
        W3, H3 = torch.empty_like(W), torch.empty_like(H)
        e2e_steps = max(3, min(args.steps, 30))
        s3 = S.Solver(M, W3, H3, alpha, mode=args.mode, precision=precision, max_iters=args.warmup + e2e_steps,
                      rule=args.rule, **kw)

        def e2e_step():
            for h, dd in zip(host_in, dev_in):
                dd.copy_(h, non_blocking=True)
            W3.copy_(hW, non_blocking=True)
            H3.copy_(hH, non_blocking=True)
            s3.run(1)
            oW.copy_(W3, non_blocking=True)
            oH.copy_(H3, non_blocking=True)
        for _ in range(min(args.warmup, 2)):
            e2e_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = max_over_ranks(pg, e0.elapsed_time(e1), dev)
        h2d = sum(t.numel() * t.element_size() for t in host_in) + 2 * hW.numel() * 4
        e2e = {"value": ws * e2e_steps / (te / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(2 * hW.numel() * 4), "steps": e2e_steps,
               "inputs": "A + W + H copied H2D from pinned memory, W + H copied D2H, every step"}
        s3.close()
    clk = clocks.stop()
    halves = st["halves"][2 * args.warmup:]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, d, ws),
            **extra,
            "lvs_stats_mean": ({"s_D": statistics.mean(h["s_D"] for h in halves),
                                "n_uniq": statistics.mean(h["n_uniq"] for h in halves), "nnz_U": nnz_u}
                               if args.mode == "lvs" and halves else None),
            "roofline": roof, "kernels": kernels, "clocks": clk, "e2e": e2e,
            "gpu_launches": kernels_per_iter * args.steps, "kernels_per_step": kernels_per_iter,
            "memsets_per_step": memsets_per_iter}
    if "exact_iters_per_s" in extra:   # LvS vs deterministic per iteration, next to the paper's CPU figure
        line["lvs_over_exact"] = {"ratio": value / extra["exact_iters_per_s"], "paper": 5.5,
                                  "paper_context": "LvS-HALS vs HALS per iteration, OAG n=37.7M k=16, 8x Xeon "
                                                   "6226 CPU, MATLAB (P:1214); context, not a target"}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, d)
    solver.close()
    return line if rank == 0 else None


def main():
    args = parse()
    ws, rank, local, pg = dist_setup(args)
    line = run_reference(args, rank, ws) if args.impl == "reference" else run_ours(args, ws, rank, local, pg)
    if line is not None and rank == 0:
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
