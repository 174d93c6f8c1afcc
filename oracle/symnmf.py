"""Plain fp64 definitions of the randomized-SymNMF hot path.

TEST INFRASTRUCTURE -- see oracle/__init__.py.  Inputs are the fp32 arrays
from synth/, promoted exactly to fp64 (O-1).  Library primitives used as
single steps: numpy matmul (BLAS dgemm), numpy.linalg.qr (Householder),
numpy.linalg.eigh, scipy.sparse CSR products.  No blocking, fusion or
reordering beyond the definitions cited.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from .philox import philox_u64, philox4x32_10, mulhi64, MASK32, S32

__all__ = [
    "as_f64", "gram", "ah", "leverage_scores", "hybrid_threshold", "fixed_point_mass",
    "draw_indices", "build_plan", "sampled_products", "hals_sweep", "hals_sweep_explicit",
    "surrogate_objective", "iterate", "gaussian_omega", "orth", "rangefinder", "lai_apply",
    "residual", "residual_fast", "nls_bruteforce", "frob_sq", "projected_gradient", "stop_index", "solve",
    "rangefinder_adaptive", "solve_lai_ir", "bpp_nnls", "bpp_update", "half_step",
]

TWO40 = float(2 ** 40)


# ----------------------------------------------------------------------- O-1
def as_f64(A):
    """O-1: promote a dense fp32 array or a CSR (rowptr/colidx/val) matrix to fp64."""
    if hasattr(A, "rowptr"):
        n = A.n
        return sp.csr_matrix((A.val.astype(np.float64), A.colidx.astype(np.int64), A.rowptr.astype(np.int64)),
                             shape=(n, n))
    if sp.issparse(A):
        return A.astype(np.float64).tocsr()
    return np.asarray(A, dtype=np.float64)


def frob_sq(A) -> float:
    """||A||_F^2 in fp64."""
    A = as_f64(A)
    if sp.issparse(A):
        return float((A.data ** 2).sum())
    return float((A * A).sum())


# ----------------------------------------------------------------------- O-2
def gram(F):
    """O-2: G = F^T F (P:420 'G_H := H^T H', P:682, P:708 CholeskyQR)."""
    F = np.asarray(F, dtype=np.float64)
    return F.T @ F


# ----------------------------------------------------------------------- O-9
def ah(A, F):
    """O-9: Y = A F, the product the paper replaces (P:181 'X H').

    A dense fp32 A is promoted to fp64 4096 rows at a time (each output row still uses its whole
    row of A; only the memory footprint changes: c5's A would be 28.8 GB in fp64)."""
    F = np.asarray(F, dtype=np.float64)
    if hasattr(A, "rowptr") or sp.issparse(A) or np.asarray(A).dtype == np.float64:
        return as_f64(A) @ F
    n = A.shape[0]
    out = np.empty((n, F.shape[1]))
    for r0 in range(0, n, 4096):
        out[r0:r0 + 4096] = np.asarray(A[r0:r0 + 4096], dtype=np.float64) @ F
    return out


# ----------------------------------------------------------------------- O-3
def leverage_scores(F):
    """O-3: l_i = ||Q[i,:]||_2^2 for Q an orthonormal basis of range(F) (Eq. 2.10).

    Computed from Householder QR (numpy.linalg.qr) -- deliberately a different
    route than the CholeskyQR the method uses; the scores are
    basis independent.
    """
    Q, _ = np.linalg.qr(np.asarray(F, dtype=np.float64), mode="reduced")
    return (Q * Q).sum(axis=1)


# ----------------------------------------------------------------------- O-4
def hybrid_threshold(lev, k: int, s: int, tau: float):
    """O-4: deterministic set of hybrid sampling.

    Reading Z1: rows with p_i = l_i/k >= tau, i.e. l_i >= T with T = tau*k
    formed once in double.  Reading Z2: s is the total budget, s_R = max(0, s - s_D).
    `lev` is the fp32 score vector the decision is taken on (promoted exactly).
    """
    l = np.asarray(lev, dtype=np.float32).astype(np.float64)
    T = float(tau) * float(k)
    det = l >= T
    det_idx = np.nonzero(det)[0]
    theta = float(l[det].sum())          # P:741 theta = sum_{I_D} l_i
    s_D = int(det_idx.size)
    s_R = max(0, int(s) - s_D)
    return {"det": det, "det_idx": det_idx, "theta": theta, "xi": float(k) - theta,
            "s_D": s_D, "s_R": s_R, "T": T}


# ----------------------------------------------------------------------- O-5
def fixed_point_mass(lev, det):
    """O-5 (readings Z3, Z6): w_i = floor(l_i * 2^40) on I_R (0 on I_D), inclusive prefix P, W = P[-1].

    p~_i = w_i / W renormalises over I_R (P:739-741 'renormalized appropriately').
    Integer arithmetic throughout (exact).
    """
    l = np.asarray(lev, dtype=np.float32).astype(np.float64)
    w = np.floor(l * TWO40).astype(np.uint64)
    w[np.asarray(det, dtype=bool)] = 0
    P = np.cumsum(w, dtype=np.uint64)
    W = int(P[-1]) if P.size else 0
    return w, P, W


# ----------------------------------------------------------------------- O-6
def draw_indices(P, W: int, s_R: int, seed: int, iteration: int, side: int):
    """O-6: s_R i.i.d. draws with replacement from p~ (P:278 'sampled with replacement').

    Reading Z6: draw j uses Philox4x32-10, counter (j lo, j hi, 2*iteration+side, 0),
    key (seed lo, seed hi); u = x1*2^32 + x0; t = floor(u*W / 2^64);
    index = first i with P_i > t (inverse CDF on the integer prefix).
    """
    if s_R <= 0 or W == 0:
        return np.empty(0, dtype=np.int64)
    j = np.arange(s_R, dtype=np.uint64)
    u, _ = philox_u64(j, 2 * int(iteration) + int(side), 0, int(seed))
    t = mulhi64(u, W)
    return np.searchsorted(P, t, side="right").astype(np.int64)


# ----------------------------------------------------------------------- O-7
def build_plan(lev, k: int, s: int, tau: float, seed: int, iteration: int, side: int):
    """O-4..O-7: the hybrid sampling plan S_H = diag(S_D, S_R) of Eq. 4.1.

    Deterministic rows carry weight 1 (S_D is a permutation); drawn
    rows carry the squared Eq. 2.11 scale 1/(s_R p~_i) = W/(s_R w_i) per draw,
    so a row drawn c_i times has omega_i = c_i * (W / (s_R * w_i)) (readings Z4, Z5),
    evaluated in IEEE double in exactly this operation order.
    """
    n = np.asarray(lev).shape[0]
    th = hybrid_threshold(lev, k, s, tau)
    w, P, W = fixed_point_mass(lev, th["det"])
    s_R = th["s_R"] if W > 0 else 0
    draws = draw_indices(P, W, s_R, seed, iteration, side)
    c = np.bincount(draws, minlength=n) if draws.size else np.zeros(n, dtype=np.int64)
    take = th["det"] | (c > 0)
    uniq = np.nonzero(take)[0]
    omega = np.empty(uniq.size, dtype=np.float64)
    for t_, i in enumerate(uniq):
        if th["det"][i]:
            omega[t_] = 1.0
        else:
            d = float(s_R) * float(int(w[i]))
            q = float(W) / d
            omega[t_] = float(int(c[i])) * q
    return {"det_idx": th["det_idx"], "draw_idx": draws, "uniq_idx": uniq, "uniq_w": omega,
            "counts": c, "s_D": th["s_D"], "s_R": s_R, "n_uniq": int(uniq.size),
            "theta": th["theta"], "xi": th["xi"], "W": W, "P": P, "w": w, "T": th["T"]}


# ----------------------------------------------------------------------- O-8
def sampled_products(A, F, uniq_idx, uniq_w):
    """O-8: G_s = F^T S^T S F and Y_s = (S A)^T (S F) (reading Z28).

    S^T S = diag(omega) on the unique rows; by symmetry row i of A is column i.
    """
    A = as_f64(A)
    F = np.asarray(F, dtype=np.float64)
    U = np.asarray(uniq_idx, dtype=np.int64)
    om = np.asarray(uniq_w, dtype=np.float64)
    FU = F[U]
    G_s = FU.T @ (om[:, None] * FU)
    AU = A[U, :]
    Y_s = AU.T @ (om[:, None] * FU)
    return np.asarray(G_s), np.asarray(Y_s)


# ----------------------------------------------------------------------- O-10
def hals_sweep(G, Y, F, X, alpha: float):
    """O-10: one sweep of the efficient symmetric HALS update, Eq. 2.6.

    For i = 1..k in order (Gauss-Seidel, reading Z9):
        x_i <- [ (Y - X G + alpha F)_i / (G_ii + alpha) + G_ii/(G_ii + alpha) x_i ]_+
    with Y = A F (or the sampled Y_s) and G = F^T F (or G_s): (A - X F^T + alpha I) f_i
    = (A F - X F^T F + alpha F)_i.  A column with G_ii + alpha = 0 is
    left unchanged.
    """
    G = np.asarray(G, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    F = np.asarray(F, dtype=np.float64)
    X = np.array(X, dtype=np.float64, copy=True)
    k = G.shape[0]
    for i in range(k):
        den = G[i, i] + alpha
        if den == 0.0:
            continue
        r = Y[:, i] - X @ G[:, i] + alpha * F[:, i]
        X[:, i] = np.maximum(r / den + (G[i, i] / den) * X[:, i], 0.0)
    return X


def hals_sweep_explicit(A, F, X, alpha: float):
    """Eq. 2.5 with the explicit residual R_i = A - sum_{j != i} x_j f_j^T.

    Test-only cross-check of hals_sweep (equivalence shown in App. A).
    Dense, O(n^2 k) memory-heavy; small n only.
    """
    A = np.asarray(as_f64(A).todense() if sp.issparse(as_f64(A)) else as_f64(A))
    F = np.asarray(F, dtype=np.float64)
    X = np.array(X, dtype=np.float64, copy=True)
    n, k = F.shape
    for i in range(k):
        R = A - X @ F.T + np.outer(X[:, i], F[:, i])
        den = F[:, i] @ F[:, i] + alpha
        if den == 0.0:
            continue
        X[:, i] = np.maximum(((R + alpha * np.eye(n)) @ F[:, i]) / den, 0.0)
    return X


def surrogate_objective(A, W, H, alpha: float) -> float:
    """Eq. 2.3: ||A - W H^T||_F^2 + alpha ||W - H||_F^2 (dense, small n)."""
    A = as_f64(A)
    A = np.asarray(A.todense()) if sp.issparse(A) else A
    W = np.asarray(W, dtype=np.float64)
    H = np.asarray(H, dtype=np.float64)
    return float(((A - W @ H.T) ** 2).sum() + alpha * ((W - H) ** 2).sum())


# ----------------------------------------------------------------------- NEXT-1 BPP
def bpp_nnls(G, b, max_iter: int = 500):
    """argmin_{x >= 0} x^T G x - 2 b^T x (G SPD) by block principal pivoting, the ANLS solver the
    paper uses (App. G; Kim & Park's full exchange with the backup rule,
    which the paper cites without restating -- SPEC S:254 accepts any exact active-set method).

    Passive set F (free variables), x_F = G_FF^{-1} b_F, dual y = G x - b on the rest;
    infeasible V = {i in F: x_i < 0} u {i not in F: y_i < 0}; exchange all of V while |V|
    shrinks (or up to 3 times without progress), else only max(V).
    """
    G = np.asarray(G, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    k = b.shape[0]
    inF = np.zeros(k, dtype=bool)
    x = np.zeros(k)
    y = -b.copy()
    ninf, p = k + 1, 3
    for _ in range(max_iter):
        V = (inF & (x < 0)) | (~inF & (y < 0))
        nv = int(V.sum())
        if nv == 0:
            break
        if nv < ninf:
            ninf, p = nv, 3
        elif p >= 1:
            p -= 1
        else:
            j = int(np.nonzero(V)[0].max())
            V = np.zeros(k, dtype=bool)
            V[j] = True
        inF = inF ^ V
        x = np.zeros(k)
        if inF.any():
            idx = np.nonzero(inF)[0]
            x[idx] = np.linalg.solve(G[np.ix_(idx, idx)], b[idx])
        y = G @ x - b
        y[inF] = 0.0
    return x


def bpp_update(G, Y, F, alpha: float):
    """Update(G + alpha I, Y + alpha F^T) by exact per-row NLS (ANLS, App. G): row r of
    the new factor solves min_{x >= 0} x^T (G + alpha I) x - 2 (Y_r + alpha F_r)^T x (bpp_nnls)."""
    G = np.asarray(G, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    F = np.asarray(F, dtype=np.float64)
    k = G.shape[0]
    Gh = G + alpha * np.eye(k)
    B = Y + alpha * F
    return np.stack([bpp_nnls(Gh, B[r]) for r in range(B.shape[0])]) if B.shape[0] else np.zeros((0, k))


# ----------------------------------------------------------------------- O-11 / O-13
def iterate(A, W0, H0, alpha: float, iters: int, mode: str = "exact", s: int = 0, tau: float = 1.0,
            seed: int = 0, first_iter: int = 0, U=None, lam=None, plans=None, record=False, rule: str = "hals"):
    """O-11 / O-13: the driver of Alg. LvS-SymNMF / LAI-SymNMF / plain HALS.

    One iteration = W-half (side 0, H fixed) then H-half (side 1, W fixed)
    (readings Z11-Z13; W0 = H0 by default in the harness).  mode:
      "exact": G = F^T F, Y = A F
      "lvs"  : scores of F (O-3) rounded to the fp32 the decision is taken in,
               plan (O-4..O-7) keyed by (seed, first_iter + t, side), G_s, Y_s (O-8);
               `plans[(it, side)]` replays a given plan instead (replay mode).
      "lai"  : G = F^T F, Y = U (Lambda (U^T F))
    then W or H <- Update(G + alpha I, Y + alpha F^T): one HALS sweep (rule "hals", Eq. 2.6)
    or the exact per-row NLS solution (rule "bpp", NEXT-1).
    Returns (W, H, trace); trace lists per-half plan statistics.
    """
    A64 = as_f64(A) if mode != "lai" else None      # LAI never touches A
    W = np.array(W0, dtype=np.float64, copy=True)
    H = np.array(H0, dtype=np.float64, copy=True)
    trace = []
    for t in range(iters):
        it = first_iter + t
        for side in (0, 1):
            W, H, st = half_step(A64, W, H, alpha, it, side, mode, s=s, tau=tau, seed=seed, U=U, lam=lam,
                                 plans=plans, record=record, rule=rule)
            trace.append(dict(it=it, side=side, **st))
    return W, H, trace


def half_step(A64, W, H, alpha: float, it: int, side: int, mode: str = "exact", s: int = 0, tau: float = 1.0,
              seed: int = 0, U=None, lam=None, plans=None, record=False, rule: str = "hals"):
    """One half of O-11 / O-13 (Alg. LvS-SymNMF lines 682-689 for side 0, 690-696 for side 1;
    LAI-SymNMF P:417-424): F = H, X = W (side 0) or F = W, X = H (side 1); X <- Update(G + alpha I,
    Y + alpha F^T).  A64 is the fp64 A of as_f64 (None for LAI).  Returns (W, H, stats)."""
    F, X = (H, W) if side == 0 else (W, H)
    k = F.shape[1]
    if mode == "exact":
        G, Y = gram(F), ah(A64, F)
        st = {}
    elif mode == "lai":
        G, Y = gram(F), lai_apply(U, lam, F)
        st = {}
    elif mode == "lvs":
        if plans is not None:
            pl = plans[(it, side)]
        else:
            lev32 = leverage_scores(F).astype(np.float32)
            pl = build_plan(lev32, k, s, tau, seed, it, side)
        G, Y = sampled_products(A64, F, pl["uniq_idx"], pl["uniq_w"])
        st = {"s_D": pl["s_D"], "s_R": pl["s_R"], "n_uniq": pl["n_uniq"], "theta": pl["theta"]}
        if record:
            st["plan"] = pl
    else:
        raise ValueError(mode)
    Xn = hals_sweep(G, Y, F, X, alpha) if rule == "hals" else bpp_update(G, Y, F, alpha)
    return (Xn, H, st) if side == 0 else (W, Xn, st)


# ----------------------------------------------------------------------- O-12
def gaussian_omega(n: int, l: int, seed: int):
    """O-12 / reading Z18: Omega (n x l, row-major element e = r*l + c) by Box-Muller on Philox.

    Pair p = e // 2 uses counter (p lo, p hi, 0, 1) (purpose 1), key (seed lo, hi):
    u1 = (x0 + 1/2) 2^-32, u2 = (x1 + 1/2) 2^-32, rho = sqrt(-2 ln u1);
    even e -> rho cos(2 pi u2), odd e -> rho sin(2 pi u2); fp64, rounded to fp32.
    """
    total = n * l
    npairs = (total + 1) // 2
    p = np.arange(npairs, dtype=np.uint64)
    x = philox4x32_10(p & MASK32, p >> S32, np.uint64(0), np.uint64(1),
                      np.uint64(seed & 0xFFFFFFFF), np.uint64((seed >> 32) & 0xFFFFFFFF))
    u1 = (x[0].astype(np.float64) + 0.5) * 2.0 ** -32
    u2 = (x[1].astype(np.float64) + 0.5) * 2.0 ** -32
    rho = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * npairs, dtype=np.float64)
    z[0::2] = rho * np.cos(2.0 * np.pi * u2)
    z[1::2] = rho * np.sin(2.0 * np.pi * u2)
    return z[:total].astype(np.float32).reshape(n, l)


def orth(Y):
    """Thin-QR orthonormal basis of range(Y) (Alg. RRF line 'thin-QR'), Householder."""
    Q, _ = np.linalg.qr(np.asarray(Y, dtype=np.float64), mode="reduced")
    return Q


def rangefinder(A, l: int, q: int, seed: int, Omega=None):
    """O-12: Alg. RRF + Alg. Apx-EVD for symmetric A.

    Y = A Omega, Q = orth(Y); q times { Y = A Q; Q = orth(Y); Y = A Q; Q = orth(Y) }
    realises (A A^T)^q A Omega with re-orthonormalisation after every application
    (reading Z16: 2q+1 applications); then T = Q^T A Q (symmetrised), T = V Lambda V^T,
    U = Q V, ordered by |lambda| descending (reading Z17).
    Returns (U, lam, Q).
    """
    n = A.n if hasattr(A, "rowptr") else A.shape[0]
    Om = gaussian_omega(n, l, seed) if Omega is None else np.asarray(Omega)
    Q = orth(ah(A, Om.astype(np.float64)))
    for _ in range(q):
        Q = orth(ah(A, Q))
        Q = orth(ah(A, Q))
    Z = ah(A, Q)
    T = Q.T @ Z
    T = 0.5 * (T + T.T)
    lam, V = np.linalg.eigh(T)
    order = np.argsort(-np.abs(lam), kind="stable")
    lam, V = lam[order], V[:, order]
    return Q @ V, lam, Q


def rangefinder_adaptive(A, l: int, q_max: int, seed: int, tol: float = 1e-3, Omega=None):
    """NEXT-2: Alg. Ada-RRF (App. E) for symmetric A, then Apx-EVD.

    Omega Gaussian (O-12); Q = qr(A Omega); then, while j <= q_max (reading Z31: j counts the
    passes of the loop, which the pseudocode never increments):
        B^T = A^T Q = A Q;  r = sqrt(||A||^2 - ||B||^2) / ||A||  (the QB residual trick)
        Q = qr(B^T)
        stop if r has decreased by no more than tol since the previous pass ("iterates
        until the normalized residual ceases to decrease by 1e-3 per power iteration") or j = q_max
        Y = A Q;  Q = qr(Y)
    Apx-EVD of the returned Q: T = Q^T A Q (symmetrised), T = V Lambda V^T, U = Q V by |lambda|.
    Returns (U, lam, Q, passes, residuals per pass).
    """
    A64 = as_f64(A)
    n = A64.shape[0]
    a2 = frob_sq(A64)
    Om = gaussian_omega(n, l, seed) if Omega is None else np.asarray(Omega)
    Q = orth(A64 @ Om.astype(np.float64))
    res = []
    j = 0
    while True:
        j += 1
        Bt = A64 @ Q
        b2 = float((Bt * Bt).sum())
        res.append(math.sqrt(max(a2 - b2, 0.0)) / math.sqrt(a2))
        Q = orth(Bt)
        if j >= q_max or (len(res) > 1 and res[-2] - res[-1] <= tol):
            break
        Q = orth(A64 @ Q)
    Z = A64 @ Q
    T = Q.T @ Z
    T = 0.5 * (T + T.T)
    lam, V = np.linalg.eigh(T)
    order = np.argsort(-np.abs(lam), kind="stable")
    lam, V = lam[order], V[:, order]
    return Q @ V, lam, Q, j, res


def solve_lai_ir(A, H0, alpha: float, U, lam, max_iters: int, tol: float = 1e-4, patience: int = 4):
    """NEXT-2 Iterative Refinement: LAI-SymNMF iterations until the stopping
    rule of P:1086 fires on the residual against the full A, then exact iterations on the full A
    from that point with the same rule.  Returns (W, H, resids LAI, resids exact)."""
    W, H, r1, d1 = solve(A, H0, alpha, max_iters, "lai", tol, patience, U=U, lam=lam)
    W2 = np.array(W, copy=True)
    H2 = np.array(H, copy=True)
    r2 = []
    for t in range(max_iters):
        W2, H2, _ = iterate(A, W2, H2, alpha, 1, "exact")
        r2.append(residual(A, H2))
        if stop_index(r2, tol, patience) is not None:
            break
    return W2, H2, r1, r2


def lai_apply(U, lam, F):
    """O-13: Y = U (Lambda (U^T F)), applied right to left (P:391-392, P:419 'replaces H^T X')."""
    U = np.asarray(U, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    F = np.asarray(F, dtype=np.float64)
    return U @ (lam[:, None] * (U.T @ F))


# ----------------------------------------------------------------------- O-14
def residual(A, H) -> float:
    """O-14: ||A - H H^T||_F / ||A||_F (Eq. 2.2; reading Z20), direct definition."""
    if not (hasattr(A, "rowptr") or sp.issparse(A)):
        # dense: rows promoted to fp64 block by block (a 60,000^2 fp32 A would be 28.8 GB in fp64)
        H = np.asarray(H, dtype=np.float64)
        n = H.shape[0]
        num = a2 = 0.0
        for r0 in range(0, n, 2048):
            blk = np.asarray(A[r0:r0 + 2048], dtype=np.float64)
            D = blk - H[r0:r0 + 2048] @ H.T
            num += float((D * D).sum())
            a2 += float((blk * blk).sum())
        return math.sqrt(num) / math.sqrt(a2)
    A64 = as_f64(A)
    H = np.asarray(H, dtype=np.float64)
    n = H.shape[0]
    if sp.issparse(A64):
        # sparse A: the exact identity ||A - H H^T||^2 = ||A||^2 - 2 tr(H^T A H) + ||H^T H||^2
        a2 = frob_sq(A64)
        G = H.T @ H
        r2 = a2 - 2.0 * float((H * (A64 @ H)).sum()) + float((G * G).sum())
        return math.sqrt(max(r2, 0.0)) / math.sqrt(a2)
    num = 0.0
    for r0 in range(0, n, 2048):
        r1 = min(n, r0 + 2048)
        blk = A64[r0:r1]
        blk = np.asarray(blk.todense()) if sp.issparse(blk) else blk
        D = blk - H[r0:r1] @ H.T
        num += float((D * D).sum())
    return math.sqrt(num) / math.sqrt(frob_sq(A64))


def residual_fast(A, W, H, AH=None) -> float:
    """App. C.2: ||A - W H^T||^2 = tr(A^T A) + tr(H W^T W H^T) - 2 tr(W^T A H), normalised."""
    A64 = as_f64(A)
    W = np.asarray(W, dtype=np.float64)
    H = np.asarray(H, dtype=np.float64)
    AH = A64 @ H if AH is None else AH
    a2 = frob_sq(A64)
    r2 = a2 + float(np.trace((W.T @ W) @ (H.T @ H))) - 2.0 * float((W * AH).sum())
    return math.sqrt(max(r2, 0.0)) / math.sqrt(a2)


# ----------------------------------------------------------------------- NEXT-3 convergence protocol
def projected_gradient(A, H):
    """Projected-gradient norm of the SymNMF objective f(H) = ||A - H H^T||_F^2 (App. D).

    grad f = 4 (H H^T - A) H, written as 4 (H (H^T H) - A H);
    (P grad)_ij = grad_ij if grad_ij < 0 or H_ij > 0, else 0 (the KKT mask).
    Returns (||P grad||_F, ||grad||_F) in fp64.
    """
    A64 = as_f64(A)
    H = np.asarray(H, dtype=np.float64)
    grad = 4.0 * (H @ (H.T @ H) - A64 @ H)
    pg = np.where((grad < 0.0) | (H > 0.0), grad, 0.0)
    return float(np.sqrt((pg * pg).sum())), float(np.sqrt((grad * grad).sum()))


def stop_index(resids, tol: float = 1e-4, patience: int = 4):
    """The experiments' stopping rule: stop once the normalised residual has failed to
    decrease by more than `tol` for `patience` consecutive iterations.  `resids[t]` is the
    residual after iteration t (t = 0, 1, ...); the decrease of iteration t is
    resids[t-1] - resids[t] (iteration 0 is compared with nothing and never counts).
    Reading Z30: "by more than 1e-4" is an absolute decrease of the normalised residual.
    Returns the number of iterations run (the stop happens after iteration t -> t + 1), or
    None if the rule never fires within the sequence.
    """
    run = 0
    for t in range(1, len(resids)):
        run = run + 1 if resids[t - 1] - resids[t] <= tol else 0
        if run >= patience:
            return t + 1
    return None


def solve(A, H0, alpha: float, max_iters: int, mode: str = "exact", tol: float = 1e-4, patience: int = 4, **kw):
    """NEXT-3 driver: iterations of `iterate` one at a time with the residual after each (O-14) and the
    stopping rule of P:1086.  Returns (W, H, resids, iterations run)."""
    W = np.array(H0, dtype=np.float64, copy=True)
    H = np.array(H0, dtype=np.float64, copy=True)
    resids = []
    first = kw.pop("first_iter", 0)
    for t in range(max_iters):
        W, H, _ = iterate(A, W, H, alpha, 1, mode, first_iter=first + t, **kw)
        resids.append(residual(A, H))
        done = stop_index(resids, tol, patience)
        if done is not None:
            return W, H, resids, done
    return W, H, resids, max_iters


# ----------------------------------------------------------------------- pins helper
def nls_bruteforce(G, y):
    """argmin_{x >= 0} x^T G x - 2 y^T x for SPD G by enumerating all 2^k passive sets (KKT check).

    The per-row QP of ANLS (App. G); test-only pin for HALS convergence (k <= 4).
    """
    G = np.asarray(G, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    k = G.shape[0]
    best, best_obj = None, np.inf
    for mask in range(1 << k):
        P = [i for i in range(k) if mask >> i & 1]
        x = np.zeros(k)
        if P:
            x[P] = np.linalg.solve(G[np.ix_(P, P)], y[P])
        if (x < -1e-14).any():
            continue
        x = np.maximum(x, 0.0)
        obj = x @ G @ x - 2 * y @ x
        if obj < best_obj:
            best, best_obj = x, obj
    return best
