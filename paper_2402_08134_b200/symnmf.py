"""Thin PyTorch binding of libsymnmf (include/symnmf.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of libsymnmf.so; PyTorch provides device memory and the current
stream.  Names follow the C ABI (symnmf_<name> -> <name>).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi as A

_PREC = {"fp32": A.FP32, "3xtf32": A.TF32X3, A.FP32: A.FP32, A.TF32X3: A.TF32X3}
_MODE = {"exact": A.EXACT, "lvs": A.LVS, "lai": A.LAI}
_RULE = {"hals": 0, "bpp": A.RULE_BPP}


def lib():
    return A.load()


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _cuda(t, dtype):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise TypeError(f"expected a contiguous CUDA {dtype} tensor")
    return t


def _workspace(fn_name, args_pre, args_post=()):
    """Run the workspace-size query, allocate, and return (ws tensor, ws ptr, size ref)."""
    fn = getattr(lib(), fn_name)
    size = C.c_size_t(0)
    A.check(fn_name, fn(*args_pre, None, C.byref(size), *args_post))
    ws = torch.empty(max(int(size.value), 256), dtype=torch.uint8, device="cuda")
    size = C.c_size_t(ws.numel())
    return ws, size


def _call(fn_name, args_pre, args_post=()):
    ws, size = _workspace(fn_name, args_pre, args_post)
    fn = getattr(lib(), fn_name)
    A.check(fn_name, fn(*args_pre, _p(ws), C.byref(size), *args_post))
    return ws


def status_of(ws) -> int:
    """Synchronise and return the device status word of a workspace."""
    out = C.c_int32(0)
    A.check("symnmf_status_read", lib().symnmf_status_read(_p(ws), C.byref(out), _stream()))
    return int(out.value)


def check_ws(ws, what=""):
    code = status_of(ws)
    if code != A.OK:
        raise A.SymNMFError(what or "device", code)


# ------------------------------------------------------------------ input matrix
class DeviceMatrix:
    """Symmetric A resident in HBM: dense fp32 n x lda, or CSR (int64 rowptr, int32 colidx, fp32 val)."""

    def __init__(self, dense=None, rowptr=None, colidx=None, val=None, n=None):
        self.dense, self.rowptr, self.colidx, self.val = dense, rowptr, colidx, val
        if dense is not None:
            _cuda(dense, torch.float32)
            self.n = dense.shape[0]
            self.kind = A.DENSE
            self.s = A.Matrix(A.DENSE, 0, self.n, dense.data_ptr(), dense.stride(0), None, None, 0)
        else:
            _cuda(rowptr, torch.int64); _cuda(colidx, torch.int32); _cuda(val, torch.float32)
            self.n = int(n if n is not None else rowptr.numel() - 1)
            self.kind = A.CSR
            self.s = A.Matrix(A.CSR, 0, self.n, val.data_ptr(), 0, rowptr.data_ptr(), colidx.data_ptr(),
                              val.numel())

    @property
    def nnz(self):
        return self.n * self.n if self.kind == A.DENSE else self.val.numel()

    @classmethod
    def from_host(cls, M, device="cuda"):
        """From a numpy dense array or a synth.CsrMatrix (rowptr/colidx/val arrays)."""
        if hasattr(M, "rowptr"):
            return cls(rowptr=torch.from_numpy(np.ascontiguousarray(M.rowptr)).to(device),
                       colidx=torch.from_numpy(np.ascontiguousarray(M.colidx)).to(device),
                       val=torch.from_numpy(np.ascontiguousarray(M.val)).to(device), n=M.n)
        return cls(dense=torch.from_numpy(np.ascontiguousarray(M, dtype=np.float32)).to(device))

    def ref(self):
        return C.byref(self.s)


# ------------------------------------------------------------------ (a1)
def gram(F: torch.Tensor) -> torch.Tensor:
    """G = F^T F (fp64), symnmf_gram."""
    _cuda(F, torch.float32)
    n, k = F.shape
    G = torch.empty((k, k), dtype=torch.float64, device=F.device)
    _call("symnmf_gram", (_p(F), n, k, _p(G)), (_stream(),))
    return G


# ------------------------------------------------------------------ (a10)
def ah(M: DeviceMatrix, F: torch.Tensor, precision="fp32", out=None) -> torch.Tensor:
    """Y = A F, symnmf_ah."""
    _cuda(F, torch.float32)
    n, k = F.shape
    Y = out if out is not None else torch.empty((n, k), dtype=torch.float32, device=F.device)
    _call("symnmf_ah", (M.ref(), _p(F), k, _p(Y), _PREC[precision]), (_stream(),))
    return Y


# ------------------------------------------------------------------ (a1-a3)
def leverage_scores(F: torch.Tensor, return_gram=False, check=True):
    """l_i = f_i (F^T F)^{-1} f_i^T by CholeskyQR, symnmf_leverage_scores."""
    _cuda(F, torch.float32)
    n, k = F.shape
    lev = torch.empty(n, dtype=torch.float32, device=F.device)
    G = torch.empty((k, k), dtype=torch.float64, device=F.device) if return_gram else None
    ws = _call("symnmf_leverage_scores", (_p(F), n, k, _p(lev), _p(G)), (_stream(),))
    if check:
        check_ws(ws, "symnmf_leverage_scores")
    return (lev, G) if return_gram else lev


# ------------------------------------------------------------------ (a4-a7)
@dataclass
class SamplingPlan:
    det_idx: torch.Tensor
    draw_idx: torch.Tensor
    uniq_idx: torch.Tensor
    uniq_w: torch.Tensor
    counts: torch.Tensor
    mass: torch.Tensor
    cap: int

    def struct(self):
        return A.Plan(self.cap, self.det_idx.data_ptr(), self.draw_idx.data_ptr(), self.uniq_idx.data_ptr(),
                      self.uniq_w.data_ptr(), self.counts.data_ptr(), self.mass.data_ptr())

    def to_host(self):
        c = self.counts.cpu().numpy()
        s_D, s_R, nu, W = (int(x) for x in c)
        m = self.mass.cpu().numpy()
        return {"det_idx": self.det_idx[:s_D].cpu().numpy().astype(np.int64),
                "draw_idx": self.draw_idx[:s_R].cpu().numpy().astype(np.int64),
                "uniq_idx": self.uniq_idx[:nu].cpu().numpy().astype(np.int64),
                "uniq_w": self.uniq_w[:nu].cpu().numpy(),
                "s_D": s_D, "s_R": s_R, "n_uniq": nu, "W": W & ((1 << 64) - 1),
                "theta": float(m[0]), "xi": float(m[1])}


def plan_from_arrays(uniq_idx, uniq_w, s_D=0, s_R=0, W=0, det_idx=None, draw_idx=None, device="cuda"):
    """A SamplingPlan holding caller-given index sets and weights (e.g. a replayed plan)."""
    uniq_idx = np.asarray(uniq_idx, dtype=np.int32)
    nu = uniq_idx.size
    det = np.asarray(det_idx if det_idx is not None else [], dtype=np.int32)
    drw = np.asarray(draw_idx if draw_idx is not None else [], dtype=np.int32)
    cap = max(nu, det.size, 1)
    pad = lambda a, m, dt: torch.from_numpy(np.concatenate([a, np.zeros(m - a.size, dtype=dt)])).to(device)
    W = int(W)
    return SamplingPlan(pad(det, cap, np.int32), pad(drw, max(drw.size, 1), np.int32), pad(uniq_idx, cap, np.int32),
                        pad(np.asarray(uniq_w, dtype=np.float64), cap, np.float64),
                        torch.tensor([s_D, s_R, nu, W - (1 << 64) if W >= (1 << 63) else W], dtype=torch.int64,
                                     device=device),
                        torch.zeros(2, dtype=torch.float64, device=device), cap)


def new_plan(n: int, s: int, cap=None, device="cuda") -> SamplingPlan:
    cap = int(cap or n)
    return SamplingPlan(torch.empty(cap, dtype=torch.int32, device=device),
                        torch.empty(max(s, 1), dtype=torch.int32, device=device),
                        torch.empty(cap, dtype=torch.int32, device=device),
                        torch.empty(cap, dtype=torch.float64, device=device),
                        torch.zeros(4, dtype=torch.int64, device=device),
                        torch.zeros(2, dtype=torch.float64, device=device), cap)


def hybrid_sample(lev: torch.Tensor, k: int, s: int, tau: float, seed: int, iteration: int, side: int,
                  cap=None, plan=None, check=True) -> SamplingPlan:
    """Hybrid deterministic + i.i.d. leverage sampling plan, symnmf_hybrid_sample."""
    _cuda(lev, torch.float32)
    n = lev.numel()
    plan = plan or new_plan(n, s, cap, lev.device)
    ps = plan.struct()
    ws = _call("symnmf_hybrid_sample", (_p(lev), n, k, s, float(tau), int(seed), int(iteration), int(side),
                                        C.byref(ps)), (_stream(),))
    if check:
        check_ws(ws, "symnmf_hybrid_sample")
    return plan


# ------------------------------------------------------------------ (a8, a9)
def sampled_ah(M: DeviceMatrix, F: torch.Tensor, plan: SamplingPlan, with_gram=True):
    """(Y_s, G_s) = ((SA)^T (SF), F^T S^T S F), symnmf_sampled_ah."""
    _cuda(F, torch.float32)
    n, k = F.shape
    Y = torch.empty((n, k), dtype=torch.float32, device=F.device)
    Gs = torch.empty((k, k), dtype=torch.float64, device=F.device) if with_gram else None
    ps = plan.struct()
    _call("symnmf_sampled_ah", (M.ref(), _p(F), k, C.byref(ps), _p(Y), _p(Gs)), (_stream(),))
    return Y, Gs


# ------------------------------------------------------------------ NEXT-4 row-sharding blocks
def leverage_scores_gram(F: torch.Tensor, G: torch.Tensor, check=True) -> torch.Tensor:
    """Scores of the rows of F given the Gram G of the whole factor, symnmf_leverage_scores_gram."""
    _cuda(F, torch.float32); _cuda(G, torch.float64)
    n, k = F.shape
    lev = torch.empty(n, dtype=torch.float32, device=F.device)
    ws = _call("symnmf_leverage_scores_gram", (_p(F), n, k, _p(G), _p(lev)), (_stream(),))
    if check:
        check_ws(ws, "symnmf_leverage_scores_gram")
    return lev


def hybrid_shard_sums(lev: torch.Tensor, k: int, tau: float):
    """(W_b, s_D_b, theta_b) of a row block's scores (host ints / float), symnmf_hybrid_shard_sums."""
    _cuda(lev, torch.float32)
    out = torch.zeros(3, dtype=torch.int64, device=lev.device)
    th = torch.zeros(1, dtype=torch.float64, device=lev.device)
    ws = _call("symnmf_hybrid_shard_sums", (_p(lev), lev.numel(), k, float(tau), C.c_void_p(out.data_ptr()),
                                            C.c_void_p(out.data_ptr() + 8), _p(th)), (_stream(),))
    check_ws(ws, "symnmf_hybrid_shard_sums")
    w, sd = (int(x) for x in out[:2].cpu().tolist())
    return w & ((1 << 64) - 1), sd, float(th.item())


def hybrid_shard_plan(lev: torch.Tensor, row0: int, k: int, s: int, tau: float, seed: int, iteration: int, side: int,
                      W_offset: int, W_total: int, sD_total: int, check=True) -> SamplingPlan:
    """The row block's part of the global plan (global row ids), symnmf_hybrid_shard_plan."""
    _cuda(lev, torch.float32)
    n = lev.numel()
    plan = new_plan(n, s, None, lev.device)
    ps = plan.struct()
    ws = _call("symnmf_hybrid_shard_plan", (_p(lev), n, int(row0), k, int(s), float(tau), int(seed), int(iteration),
                                            int(side), C.c_uint64(int(W_offset)), C.c_uint64(int(W_total)),
                                            int(sD_total), C.byref(ps)), (_stream(),))
    if check:
        check_ws(ws, "symnmf_hybrid_shard_plan")
    return plan


def plan_rows_scaled(F: torch.Tensor, row0: int, plan: SamplingPlan, with_gram=True):
    """(Z, G_s part) for a row block's plan rows, symnmf_plan_rows_scaled."""
    _cuda(F, torch.float32)
    k = F.shape[1]
    Z = torch.empty((plan.cap, k), dtype=torch.float32, device=F.device)
    Gs = torch.empty((k, k), dtype=torch.float64, device=F.device) if with_gram else None
    ps = plan.struct()
    _call("symnmf_plan_rows_scaled", (_p(F), int(row0), k, C.byref(ps), _p(Z), _p(Gs)), (_stream(),))
    return Z, Gs


def sampled_ah_rows(Mb: DeviceMatrix, n_total: int, uniq: torch.Tensor, Z: torch.Tensor, k: int) -> torch.Tensor:
    """Rows of the sampled product for a CSR row block (pull form), symnmf_sampled_ah_rows."""
    _cuda(uniq, torch.int32); _cuda(Z, torch.float32)
    nu = torch.tensor([uniq.numel()], dtype=torch.int64, device=Z.device)
    Y = torch.empty((Mb.n, k), dtype=torch.float32, device=Z.device)
    _call("symnmf_sampled_ah_rows", (Mb.ref(), int(n_total), _p(uniq), _p(nu), max(uniq.numel(), 1), _p(Z), k, _p(Y)),
          (_stream(),))
    return Y


def lai_project_rows(U: torch.Tensor, F: torch.Tensor) -> torch.Tensor:
    """Z_b = U_b^T F_b (fp64 l x k) of a row block, symnmf_lai_project_rows."""
    _cuda(U, torch.float32); _cuda(F, torch.float32)
    n, l = U.shape
    k = F.shape[1]
    Z = torch.empty((l, k), dtype=torch.float64, device=F.device)
    _call("symnmf_lai_project_rows", (_p(U), n, l, _p(F), k, _p(Z)), (_stream(),))
    return Z


def lai_apply_rows(U: torch.Tensor, lam: torch.Tensor, Z: torch.Tensor) -> torch.Tensor:
    """Y_b = U_b (Lambda Z) (fp32 n_b x k) of a row block, symnmf_lai_apply_rows."""
    _cuda(U, torch.float32); _cuda(lam, torch.float64); _cuda(Z, torch.float64)
    n, l = U.shape
    k = Z.shape[1]
    Y = torch.empty((n, k), dtype=torch.float32, device=U.device)
    _call("symnmf_lai_apply_rows", (_p(U), _p(lam), n, l, _p(Z), k, _p(Y)), (_stream(),))
    return Y


# ------------------------------------------------------------------ (a12, a13)
def gaussian(n: int, l: int, seed: int, device="cuda") -> torch.Tensor:
    Om = torch.empty((n, l), dtype=torch.float32, device=device)
    A.check("symnmf_gaussian", lib().symnmf_gaussian(n, l, int(seed), _p(Om), _stream()))
    return Om


def rangefinder(M: DeviceMatrix, l: int, q: int, seed: int, precision="fp32", check=True):
    """(U, lambda) of Alg. RRF + Apx-EVD, symnmf_rangefinder."""
    U = torch.empty((M.n, l), dtype=torch.float32, device="cuda")
    lam = torch.empty(l, dtype=torch.float64, device="cuda")
    ws = _call("symnmf_rangefinder", (M.ref(), l, q, int(seed), _PREC[precision], _p(U), _p(lam)), (_stream(),))
    if check:
        check_ws(ws, "symnmf_rangefinder")
    return U, lam


def rangefinder_adaptive(M: DeviceMatrix, l: int, q_max: int, seed: int, tol: float = 1e-3, precision="fp32"):
    """(U, lambda, passes, residual per pass) of Alg. Ada-RRF + Apx-EVD, symnmf_rangefinder_adaptive."""
    U = torch.empty((M.n, l), dtype=torch.float32, device="cuda")
    lam = torch.empty(l, dtype=torch.float64, device="cuda")
    passes = C.c_int32(0)
    res = (C.c_double * q_max)()
    _call("symnmf_rangefinder_adaptive", (M.ref(), l, q_max, float(tol), int(seed), _PREC[precision], _p(U), _p(lam),
                                          C.byref(passes), res), (_stream(),))
    return U, lam, passes.value, [res[i] for i in range(passes.value)]


def lai_ah(U: torch.Tensor, lam: torch.Tensor, F: torch.Tensor) -> torch.Tensor:
    """Y = U (Lambda (U^T F)), symnmf_lai_ah."""
    _cuda(U, torch.float32); _cuda(lam, torch.float64); _cuda(F, torch.float32)
    n, l = U.shape
    k = F.shape[1]
    Y = torch.empty((n, k), dtype=torch.float32, device=F.device)
    _call("symnmf_lai_ah", (_p(U), _p(lam), n, l, _p(F), k, _p(Y)), (_stream(),))
    return Y


# ------------------------------------------------------------------ (a11)
def hals_sweep(G: torch.Tensor, Y: torch.Tensor, F: torch.Tensor, X: torch.Tensor, alpha: float,
               return_gram=False):
    """One sweep of Update(G + alpha I, Y + alpha F^T) on X (in place), symnmf_hals_sweep."""
    _cuda(G, torch.float64); _cuda(Y, torch.float32); _cuda(F, torch.float32); _cuda(X, torch.float32)
    n, k = X.shape
    Gn = torch.empty((k, k), dtype=torch.float64, device=X.device) if return_gram else None
    _call("symnmf_hals_sweep", (_p(G), _p(Y), _p(F), _p(X), n, k, float(alpha), _p(Gn)), (_stream(),))
    return (X, Gn) if return_gram else X


def bpp_update(G: torch.Tensor, Y: torch.Tensor, F: torch.Tensor, X: torch.Tensor, alpha: float,
               return_gram=False):
    """X <- exact per-row NLS with (G + alpha I, Y + alpha F^T) by block principal pivoting,
    symnmf_bpp_update.  Returns X (and X^T X if return_gram) and the non-converged row count."""
    _cuda(G, torch.float64); _cuda(Y, torch.float32); _cuda(F, torch.float32); _cuda(X, torch.float32)
    n, k = X.shape
    Gn = torch.empty((k, k), dtype=torch.float64, device=X.device) if return_gram else None
    nc = C.c_int32(0)
    _call("symnmf_bpp_update", (_p(G), _p(Y), _p(F), _p(X), n, k, float(alpha), _p(Gn), C.byref(nc)), (_stream(),))
    return (X, Gn, nc.value) if return_gram else (X, nc.value)


# ------------------------------------------------------------------ (a15)
def residual(M: DeviceMatrix, H: torch.Tensor) -> torch.Tensor:
    """[||A - H H^T|| / ||A||, ||A||^2, tr(H^T A H), ||H^T H||^2] (fp64, device), symnmf_residual."""
    _cuda(H, torch.float32)
    out = torch.empty(4, dtype=torch.float64, device=H.device)
    _call("symnmf_residual", (M.ref(), _p(H), H.shape[1], _p(out)), (_stream(),))
    return out


def projected_gradient(M: DeviceMatrix, H: torch.Tensor, precision: str = "fp32") -> torch.Tensor:
    """[||P grad f||_F, ||grad f||_F] of f(H) = ||A - H H^T||^2 (fp64, device), symnmf_projected_gradient."""
    _cuda(H, torch.float32)
    out = torch.empty(2, dtype=torch.float64, device=H.device)
    _call("symnmf_projected_gradient", (M.ref(), _p(H), H.shape[1], _PREC[precision], _p(out)), (_stream(),))
    return out


# ------------------------------------------------------------------ (a14)
class Solver:
    """Captured-graph iteration driver (symnmf_solver_*)."""

    def __init__(self, M, W, H, alpha, mode="exact", precision="fp32", s=0, tau=1.0, seed=0, first_iter=0,
                 max_iters=1, U=None, lam=None, with_residual=False, rule="hals", record_plans=False):
        _cuda(W, torch.float32); _cuda(H, torch.float32)
        n, k = H.shape
        self.M, self.W, self.H, self.U, self.lam = M, W, H, U, lam
        self.max_iters = max_iters
        l = U.shape[1] if U is not None else 0
        mref = M.ref() if M is not None else None
        flags = _MODE[mode] | _RULE[rule] | (A.RECORD_PLANS if record_plans else 0)
        pre = (mref, n, _p(W), _p(H), k, float(alpha), flags, _PREC[precision], int(s), float(tau),
               int(seed), int(first_iter), int(max_iters), _p(U), _p(lam), l, 1 if with_residual else 0)
        fn = lib().symnmf_solver_create
        size = C.c_size_t(0)
        A.check("symnmf_solver_create", fn(None, *pre, None, C.byref(size), _stream()))
        self.ws = torch.empty(max(int(size.value), 256), dtype=torch.uint8, device="cuda")
        size = C.c_size_t(self.ws.numel())
        self.h = C.c_void_p()
        A.check("symnmf_solver_create", fn(C.byref(self.h), *pre, _p(self.ws), C.byref(size), _stream()))

    def run(self, iters: int):
        A.check("symnmf_solver_run", lib().symnmf_solver_run(self.h, int(iters), _stream()))

    def run_until(self, max_iters: int, tol: float = 1e-4, patience: int = 4) -> int:
        """NEXT-3 stopping rule: iterate until the residual fails to decrease by more than
        `tol` for `patience` consecutive iterations (needs with_residual=True).  Returns iterations run."""
        done = C.c_int32(0)
        A.check("symnmf_solver_run_until", lib().symnmf_solver_run_until(self.h, int(max_iters), float(tol),
                                                                         int(patience), C.byref(done), _stream()))
        return done.value

    def pgrad(self):
        """Projected-gradient norms ||P grad f(H)||_F after each recorded iteration (with_residual=True)."""
        m = self.max_iters
        buf = (C.c_double * m)()
        A.check("symnmf_solver_pgrad", lib().symnmf_solver_pgrad(self.h, buf, _stream()))
        done = self.stats()["iters"]
        return [buf[i] for i in range(min(done, m))]

    def last_plan(self):
        """(scores, plan) the LvS solver drew in the last half it ran, copied on the current stream
        (symnmf_solver_last_plan); det_idx / draw_idx are not materialised by the fused sampler."""
        n, dev = self.W.shape[0], self.W.device
        lev = torch.empty(n, dtype=torch.float32, device=dev)
        plan = SamplingPlan(torch.empty(0, dtype=torch.int32, device=dev), torch.empty(0, dtype=torch.int32, device=dev),
                            torch.empty(n, dtype=torch.int32, device=dev), torch.empty(n, dtype=torch.float64, device=dev),
                            torch.empty(4, dtype=torch.int64, device=dev), torch.empty(2, dtype=torch.float64, device=dev),
                            n)
        A.check("symnmf_solver_last_plan",
                lib().symnmf_solver_last_plan(self.h, _p(lev), _p(plan.uniq_idx), _p(plan.uniq_w), _p(plan.counts),
                                              _p(plan.mass), _stream()))
        return lev, plan

    def plan_history(self, t: int, side: int):
        """(scores, plan) the LvS solver drew in half `side` of its iteration t (created with
        record_plans=True; symnmf_solver_plan_history)."""
        n, dev = self.W.shape[0], self.W.device
        lev = torch.empty(n, dtype=torch.float32, device=dev)
        plan = SamplingPlan(torch.empty(0, dtype=torch.int32, device=dev), torch.empty(0, dtype=torch.int32, device=dev),
                            torch.empty(n, dtype=torch.int32, device=dev), torch.empty(n, dtype=torch.float64, device=dev),
                            torch.empty(4, dtype=torch.int64, device=dev), torch.empty(2, dtype=torch.float64, device=dev),
                            n)
        A.check("symnmf_solver_plan_history",
                lib().symnmf_solver_plan_history(self.h, int(t), int(side), _p(lev), _p(plan.uniq_idx),
                                                 _p(plan.uniq_w), _p(plan.counts), _p(plan.mass), _stream()))
        return lev, plan

    def stats(self):
        m = self.max_iters
        st = (A.HalfStats * (2 * m))()
        rs = (C.c_double * m)()
        done = C.c_int32(0)
        code = lib().symnmf_solver_stats(self.h, C.byref(done), st, rs, _stream())
        k = min(done.value, m)
        halves = [{"s_D": st[i].s_d, "s_R": st[i].s_r, "n_uniq": st[i].n_uniq, "theta": st[i].theta}
                  for i in range(2 * k)]
        return {"status": code, "iters": done.value, "halves": halves, "residual": [rs[i] for i in range(k)]}

    def profile(self, iters=5):
        """Per launch site of one iteration: [(name, mean ms)], from eager evented iterations."""
        cap = 64
        names = C.create_string_buffer(48 * cap)
        ms = (C.c_float * cap)()
        cnt = C.c_int32(0)
        A.check("symnmf_solver_profile", lib().symnmf_solver_profile(self.h, int(iters), cap, names, ms,
                                                                     C.byref(cnt), _stream()))
        raw = names.raw
        out = []
        for i in range(cnt.value):
            nm = raw[48 * i:48 * (i + 1)].split(b"\0", 1)[0].decode()
            out.append((nm, float(ms[i])))
        return out

    def graph_nodes(self):
        kc, mc = C.c_int32(0), C.c_int32(0)
        A.check("symnmf_solver_graph_nodes", lib().symnmf_solver_graph_nodes(self.h, C.byref(kc), C.byref(mc)))
        return int(kc.value), int(mc.value)

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().symnmf_solver_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def iterate(M, W, H, alpha, iters, mode="exact", precision="fp32", s=0, tau=1.0, seed=0, first_iter=0, U=None,
            lam=None, with_residual=False, rule="hals"):
    """symnmf_iterate: `iters` iterations in place on (W, H); returns stats and residual trace."""
    _cuda(W, torch.float32); _cuda(H, torch.float32)
    n, k = H.shape
    l = U.shape[1] if U is not None else 0
    st = (A.HalfStats * (2 * iters))()
    rs = (C.c_double * iters)()
    pre = (M.ref() if M is not None else None, n, _p(W), _p(H), k, float(alpha), _MODE[mode] | _RULE[rule],
           _PREC[precision], int(s), float(tau), int(seed), int(first_iter), int(iters), _p(U), _p(lam), l, st,
           rs if with_residual else None)
    ws = _call("symnmf_iterate", pre, (_stream(),))
    del ws
    halves = [{"s_D": st[i].s_d, "s_R": st[i].s_r, "n_uniq": st[i].n_uniq, "theta": st[i].theta}
              for i in range(2 * iters)]
    return {"halves": halves, "residual": list(rs) if with_residual else None}


def solve(M, W, H, alpha, max_iters, mode="exact", precision="fp32", s=0, tau=1.0, seed=0, U=None, lam=None,
          tol=1e-4, patience=4, refine=False, rule="hals"):
    """symnmf_solve: iterate until the P:1086 stopping rule; refine=True adds Iterative Refinement
    (EXACT on the full A after LAI).  Returns {"iters": [phase0, phase1], "residual": [list, list]}."""
    _cuda(W, torch.float32); _cuda(H, torch.float32)
    n, k = H.shape
    l = U.shape[1] if U is not None else 0
    its = (C.c_int32 * 2)()
    rs = (C.c_double * (2 * max_iters))()
    pre = (M.ref() if M is not None else None, n, _p(W), _p(H), k, float(alpha), _MODE[mode] | _RULE[rule],
           _PREC[precision], int(s), float(tau), int(seed), _p(U), _p(lam), l, int(max_iters), float(tol), int(patience),
           1 if refine else 0, its, rs)
    ws = _call("symnmf_solve", pre, (_stream(),))
    del ws
    return {"iters": [its[0], its[1]],
            "residual": [[rs[i] for i in range(its[0])], [rs[max_iters + i] for i in range(its[1])]]}
