#!/usr/bin/env python
"""Benchmark of the randomized-SymNMF hot path on B200 (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--mode lvs] [--impl ours|reference]

A step is one full LvS-HALS iteration (W-half + H-half: Gram, CholeskyQR
scores, hybrid plan, sampled Gram, sampled product, HALS sweep) of config
`--config` (default configs[1] = c2), replayed from the solver's captured
CUDA graph with inputs resident in HBM.  L2 is flushed (256 MiB write)
before every timed step.  N > 1 runs N independent replicas (DESIGN.md §7:
the single-GPU north star does not shard; weak scaling, no collective on
the data path), timed on the device as the max over ranks.
"""
import argparse
import json
import math
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
SLEEP_CYCLES = 400_000   # ~0.2 ms: hides host enqueue latency from the device-side event timing


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--mode", default="lvs", choices=["lvs", "exact"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="warmup + timed loop only (for ncu)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


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
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
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
        rows = self.rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
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
        backend = "nccl" if args.impl == "ours" else "gloo"
        if args.impl == "ours":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        pg = dist
    return ws, rank, local, pg


# ------------------------------------------------------------------ algorithmic bytes
def kernel_bytes(name, n, k, nnz_u=0, n_u=0, nnz=0):
    if name == "sampled_ah_csr":          # 8 nnz_U + 16|U| + 4|U|k gathered + 4nk output write
        return 8 * nnz_u + 16 * n_u + 4 * n_u * k + 4 * n * k
    if name == "hals_sweep":              # read Y, X, F + write X
        return 16 * n * k
    if name == "gram":
        return 4 * n * k
    if name == "leverage":
        return 4 * n * k + 4 * n
    if name == "spmm_csr":                # 8 nnz + 8(n+1) + 4nk (F once) + 4nk (Y)
        return 8 * nnz + 8 * (n + 1) + 8 * n * k
    if name == "hybrid_sample":           # lev read x3, P u64 write+searches, counts, plan
        return 4 * n * 3 + 8 * n + 4 * n * 2
    raise KeyError(name)


# ------------------------------------------------------------------ reference arm: the oracle on host cores
def run_reference(args, rank, ws):
    import numpy as np
    import oracle as O
    from synth import make_input
    if rank != 0:
        return None
    d = make_input(args.config)
    cfg = d["cfg"]
    A, H0, alpha = d["A"], d["H0"], d["alpha"]
    kw = dict(s=cfg.s, tau=cfg.tau, seed=0) if args.mode == "lvs" else {}
    W, H = H0.astype(np.float64), H0.astype(np.float64)
    it = 0
    for _ in range(args.warmup):
        W, H, _ = O.iterate(A, W, H, alpha, 1, args.mode, first_iter=it, **kw)
        it += 1
    t0 = time.perf_counter()
    for _ in range(args.steps):
        W, H, _ = O.iterate(A, W, H, alpha, 1, args.mode, first_iter=it, **kw)
        it += 1
    dt = time.perf_counter() - t0
    v = args.steps / dt
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n": d["n"], "k": cfg.k, "mode": args.mode,
                       "s": cfg.s, "tau": cfg.tau},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} full oracle {args.mode} iterations of {args.config}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def cpu_baseline(args, budget_s=15.0):
    import numpy as np
    import oracle as O
    from synth import make_input
    d = make_input(args.config)
    cfg = d["cfg"]
    kw = dict(s=cfg.s, tau=cfg.tau, seed=0) if args.mode == "lvs" else {}
    W = H = d["H0"].astype(np.float64)
    t0 = time.perf_counter()
    done = 0
    while True:
        W, H, _ = O.iterate(d["A"], W, H, d["alpha"], 1, args.mode, first_iter=done, **kw)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"first {done} oracle {args.mode} iterations of {args.config} (full n), ~{budget_s:.0f} s budget"}


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
    M = S.DeviceMatrix.from_host(A)
    W = torch.from_numpy(H0).to(dev)
    H = torch.from_numpy(H0).to(dev)
    lvs = args.mode == "lvs"
    kw = dict(s=cfg.s, tau=cfg.tau, seed=cfg.seed) if lvs else {}
    total = args.warmup + args.steps
    solver = S.Solver(M, W, H, alpha, mode=args.mode, max_iters=total, **kw)
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
        torch.cuda._sleep(SLEEP_CYCLES)   # keep the GPU busy while the host enqueues the step
        e0.record(stream)
        solver.run(1)
        e1.record(stream)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    t_ms = sum(step_ms)
    st = solver.stats()
    if st["status"] != 0:
        raise RuntimeError(f"device status {st['status']}")
    kernels_per_iter, memsets_per_iter = solver.graph_nodes()
    if args.profile_only:
        clocks.stop()
        return None
    t_max = t_ms
    if pg:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        t_max = float(tt.item())
    value = ws * args.steps / (t_max / 1e3)

    # exact-product iterations (the "exact" half of the metric), same protocol
    ex_steps = max(3, min(args.steps, 30))
    W2 = torch.from_numpy(H0).to(dev)
    H2 = torch.from_numpy(H0).to(dev)
    sx = S.Solver(M, W2, H2, alpha, mode="exact", max_iters=args.warmup + ex_steps)
    sx.run(args.warmup)
    torch.cuda.synchronize()
    ex_ms = []
    for _ in range(ex_steps):
        flush.zero_()
        torch.cuda._sleep(SLEEP_CYCLES)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); sx.run(1); e1.record(stream)
        e1.synchronize()
        ex_ms.append(e0.elapsed_time(e1))
    exact_ips = ex_steps / (sum(ex_ms) / 1e3)

    # per-kernel phase timing on the same inputs (eager ABI calls, CUDA events on this stream)
    F = H.clone()
    X = W.clone()
    reps = 20
    def timeit(fn):
        fn(); torch.cuda.synchronize()
        acc = 0.0
        for _ in range(reps):
            flush.zero_()
            torch.cuda._sleep(SLEEP_CYCLES)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream); fn(); e1.record(stream)
            e1.synchronize()
            acc += e0.elapsed_time(e1)
        return acc / reps
    lev = S.leverage_scores(F)
    phases = {"gram": timeit(lambda: S.gram(F)), "leverage": timeit(lambda: S.leverage_scores(F, check=False))}
    if lvs:
        plan = S.hybrid_sample(lev, k, cfg.s, cfg.tau, 0, 0, 0)
        phases["hybrid_sample"] = timeit(lambda: S.hybrid_sample(lev, k, cfg.s, cfg.tau, 0, 0, 0, plan=plan,
                                                                 check=False))
        Y, Gs = S.sampled_ah(M, F, plan)
        phases["sampled_ah_csr" if M.kind == 1 else "sampled_ah_dense"] = timeit(lambda: S.sampled_ah(M, F, plan))
        ph = plan.to_host()
        rp = A.rowptr if hasattr(A, "rowptr") else None
        nnz_u = int(sum(rp[i + 1] - rp[i] for i in ph["uniq_idx"])) if rp is not None else 0
        n_u = ph["n_uniq"]
    else:
        Y = S.ah(M, F)
        phases["spmm_csr"] = timeit(lambda: S.ah(M, F, out=Y))
        nnz_u = n_u = 0
    G = S.gram(F)
    phases["hals_sweep"] = timeit(lambda: S.hals_sweep(G, Y, F, X, alpha))
    dom = max(phases, key=phases.get)
    pk, which = peaks()
    nnz = A.nnz if hasattr(A, "nnz") else n * n
    try:
        algo = kernel_bytes(dom, n, k, nnz_u=nnz_u, n_u=n_u, nnz=nnz)
    except KeyError:
        algo = None
    achieved = algo / (phases[dom] * 1e-3) / 1e9 if algo else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": (achieved / pk["hbm_gbs"]) if achieved else None, "traffic": traffic,
                "algorithmic_bytes": algo, "kernel_ms": phases[dom], "peak_source": which,
                "phases_ms": {kk: round(v, 5) for kk, v in phases.items()}}

    # end to end through the public API: pinned host inputs in, result out, every step
    e2e = None
    if not args.no_e2e:
        if hasattr(A, "rowptr"):
            host_in = [torch.from_numpy(A.rowptr).pin_memory(), torch.from_numpy(A.colidx).pin_memory(),
                       torch.from_numpy(A.val).pin_memory()]
            dev_in = [M.rowptr, M.colidx, M.val]
        else:
            host_in = [torch.from_numpy(A).pin_memory()]
            dev_in = [M.dense]
        hW = torch.from_numpy(H0).pin_memory(); hH = torch.from_numpy(H0).pin_memory()
        oW = torch.empty_like(hW).pin_memory(); oH = torch.empty_like(hH).pin_memory()
        W3 = torch.empty_like(W); H3 = torch.empty_like(H)
        s3 = S.Solver(M, W3, H3, alpha, mode=args.mode, max_iters=args.warmup + args.steps, **kw)
        def e2e_step():
            for h, dd in zip(host_in, dev_in):
                dd.copy_(h, non_blocking=True)
            W3.copy_(hW, non_blocking=True); H3.copy_(hH, non_blocking=True)
            s3.run(1)
            oW.copy_(W3, non_blocking=True); oH.copy_(H3, non_blocking=True)
        for _ in range(args.warmup):
            e2e_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1)
        if pg:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            pg.all_reduce(tt, op=pg.ReduceOp.MAX)
            te = float(tt.item())
        h2d = sum(t.numel() * t.element_size() for t in host_in) + 2 * hW.numel() * 4
        e2e = {"value": ws * args.steps / (te / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 2 * hW.numel() * 4}
    clk = clocks.stop()
    halves = st["halves"][2 * args.warmup:]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "n": n, "nnz": int(nnz), "k": k, "mode": args.mode,
                       "s": cfg.s if lvs else None, "tau": cfg.tau if lvs else None,
                       "l2": "flushed (256 MiB write) before every timed step", "parallelism": f"replicas{ws}",
                       "graph": "per-iteration CUDA graph replay"},
            "exact_iters_per_s": exact_ips * ws,
            "lvs_stats_mean": {"s_D": statistics.mean(h["s_D"] for h in halves) if halves else None,
                               "n_uniq": statistics.mean(h["n_uniq"] for h in halves) if halves else None},
            "roofline": roofline, "clocks": clk, "e2e": e2e,
            "gpu_launches": kernels_per_iter * args.steps, "kernels_per_step": kernels_per_iter,
            "memsets_per_step": memsets_per_iter}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    solver.close(); sx.close()
    return line if rank == 0 else None


def main():
    args = parse()
    ws, rank, local, pg = dist_setup(args)
    if args.impl == "reference":
        line = run_reference(args, rank, ws)
    else:
        line = run_ours(args, ws, rank, local, pg)
    if line is not None and rank == 0:
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
