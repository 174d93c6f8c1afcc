"""The five BASELINE.json configurations as seeded synthetic inputs.

Recipes follow SURVEY.md §8(d) ("Generation rules" and the per-config table);
DESIGN.md §3 restates them.  RNG: numpy Generator(PCG64) seeded through
SeedSequence(seed).spawn(2): stream 0 draws the data matrix, stream 1 the
initial factor.  Everything returned is what BOTH the CUDA path and the oracle
consume; nothing here computes any step of SymNMF itself.

Stand-ins: the paper's WoS (dense EDVW adjacency)
and OAG (sparse citation graph) datasets are absent; c3/c5 stand
in for dense similarity graphs, c2/c4 for large sparse graphs.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    k: int
    kind: str            # "dense" | "csr"
    s: int               # LvS sample budget (total, reading Z2)
    tau: float           # hybrid threshold on p_i = l_i / k (reading Z1)
    iters: int
    modes: tuple
    seed: int = 0
    l: int = 0           # LAI sketch width (k + rho)
    q: int = 0           # LAI power iterations
    note: str = ""


CONFIGS = {
    "c1": Config("c1", 1_000, 8, "dense", 200, 1.0 / 200, 20, ("exact", "lvs"),
                 note="planted 8 blocks + |N(0,0.01)| noise"),
    "c2": Config("c2", 100_000, 16, "csr", 2_000, 1.0 / 2_000, 30, ("exact", "lvs"),
                 note="SBM 16 communities, ~18 intra / ~2 inter degree"),
    "c3": Config("c3", 30_000, 32, "dense", 3_000, 1.0 / 3_000, 30, ("exact", "lvs"),
                 note="Gaussian kernel on 64-dim 32-component mixture"),
    "c4": Config("c4", 2_000_000, 32, "csr", 20_000, 1.0 / 20_000, 20, ("exact", "lvs"),
                 note="power-law (exp 2.5) 32-community graph, ~100M nnz"),
    "c5": Config("c5", 60_000, 64, "dense", 0, 0.0, 50, ("lai",), l=74, q=2,
                 note="Gaussian kernel on 128-dim 64-component mixture, LAI"),
}


@dataclass
class CsrMatrix:
    """Symmetric sparse matrix, both triangles stored, rows sorted."""
    n: int
    rowptr: np.ndarray   # int64 [n+1]
    colidx: np.ndarray   # int32 [nnz], sorted within each row, unique
    val: np.ndarray      # float32 [nnz]
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n), dtype=np.float32)
        rows = np.repeat(np.arange(self.n), np.diff(self.rowptr))
        out[rows, self.colidx] = self.val
        return out


def _streams(seed: int):
    data_ss, init_ss = np.random.SeedSequence(seed).spawn(2)
    return np.random.Generator(np.random.PCG64(data_ss)), np.random.Generator(np.random.PCG64(init_ss))


# ---------------------------------------------------------------- c1: planted
def planted_dense(n: int, k: int, noise_std: float, rng: np.random.Generator):
    """A = H0 H0^T + (E + E^T)/2, E_ij = |N(0, noise_std^2)| (reading Z22: std).

    H0 rows are one-hot on cluster g_i = floor(k i / n) with U(0.5, 1) values.
    Returns (A fp32 exactly symmetric, H0 fp64).
    """
    g = (k * np.arange(n)) // n
    H0 = np.zeros((n, k))
    H0[np.arange(n), g] = rng.uniform(0.5, 1.0, size=n)
    A = H0 @ H0.T
    if noise_std > 0:
        E = np.abs(rng.normal(0.0, noise_std, size=(n, n)))
        A = A + (E + E.T) / 2.0
    A32 = A.astype(np.float32)
    return A32, H0


# ---------------------------------------------------------------- CSR helpers
def _build_csr(n: int, u: np.ndarray, v: np.ndarray, w: np.ndarray, meta: dict) -> CsrMatrix:
    """Mirror undirected edges (u < v, unique) into a symmetric CSR matrix."""
    rows = np.concatenate([u, v]).astype(np.int64)
    cols = np.concatenate([v, u]).astype(np.int64)
    vals = np.concatenate([w, w]).astype(np.float32)
    order = np.argsort(rows * n + cols, kind="stable")
    rows, cols, vals = rows[order], cols[order], vals[order]
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rowptr[1:])
    return CsrMatrix(n, rowptr, cols.astype(np.int32), vals, meta)


def _relabel(n, u, v, rng):
    perm = rng.permutation(n)
    a, b = perm[u], perm[v]
    return np.minimum(a, b), np.maximum(a, b)


# ---------------------------------------------------------------- c2: SBM
def sbm_csr(n: int, n_comm: int, deg_in: float, deg_out: float, rng: np.random.Generator) -> CsrMatrix:
    """Stochastic block model: per block pair a Binomial edge count over the
    upper-triangle pairs, uniform positions, duplicates collapsed, weights in
    (0, 1], zero diagonal, seeded vertex relabel."""
    m = n // n_comm
    p_in = deg_in / (m - 1)
    p_out = deg_out / (n - m)
    # block a holds rows [a m, a m + sz[a]); the last block absorbs the n % n_comm remainder
    # (identical draws to equal blocks when n_comm divides n)
    sz = [m] * (n_comm - 1) + [n - (n_comm - 1) * m]
    keys = []
    for a in range(n_comm):
        for b in range(a, n_comm):
            if a == b:
                cnt = rng.binomial(sz[a] * (sz[a] - 1) // 2, p_in)
                i = rng.integers(0, sz[a], cnt) + a * m
                j = rng.integers(0, sz[a], cnt) + a * m
            else:
                cnt = rng.binomial(sz[a] * sz[b], p_out)
                i = rng.integers(0, sz[a], cnt) + a * m
                j = rng.integers(0, sz[b], cnt) + b * m
            keep = i != j
            i, j = i[keep], j[keep]
            keys.append(np.minimum(i, j).astype(np.int64) * n + np.maximum(i, j))
    key = np.unique(np.concatenate(keys))
    u, v = key // n, key % n
    w = (1.0 - rng.random(key.size)).astype(np.float32)
    u, v = _relabel(n, u, v, rng)
    return _build_csr(n, u, v, w, {"generator": "sbm", "communities": n_comm,
                                   "p_in": p_in, "p_out": p_out})


# ---------------------------------------------------------------- c4: power law
def powerlaw_csr(n: int, n_comm: int, mean_deg: float, tail: float, mix: float,
                 rng: np.random.Generator) -> CsrMatrix:
    """Chung-Lu style power-law community graph (reading Z24).

    theta_i = U^{-1/tail} (Pareto tail 1.5 <=> degree exponent 2.5), rescaled to
    mean `mean_deg`, capped at sqrt(sum theta).  Exactly n*mean_deg/2 unique
    undirected edges are kept: endpoint u ~ theta; with prob 1-mix v ~ theta
    inside u's community, else v ~ theta globally; self loops dropped,
    duplicates collapsed, draws topped up.  Weights 1-U[0,1); vertex relabel.
    """
    m = n // n_comm
    theta = (1.0 - rng.random(n)) ** (-1.0 / tail)
    theta *= mean_deg / theta.mean()
    theta = np.minimum(theta, math.sqrt(theta.sum()))
    cum = np.cumsum(theta)
    total = cum[-1]
    # community c = rows [c m, last[c]]; the last one absorbs the n % n_comm remainder (identical
    # to equal communities when n_comm divides n)
    last = np.minimum(np.arange(1, n_comm + 1) * m, n) - 1
    last[-1] = n - 1
    comm_end = cum[last]
    comm_start = np.concatenate([[0.0], comm_end[:-1]])
    comm_mass = comm_end - comm_start
    target = int(n * mean_deg) // 2
    have = np.empty(0, dtype=np.int64)
    while have.size < target:
        B = int((target - have.size) * 1.08) + 1024
        u = np.searchsorted(cum, rng.random(B) * total, side="right")
        u = np.minimum(u, n - 1)
        inter = rng.random(B) < mix
        c = np.minimum(u // m, n_comm - 1)
        x = np.where(inter, rng.random(B) * total, comm_start[c] + rng.random(B) * comm_mass[c])
        v = np.searchsorted(cum, x, side="right")
        v = np.minimum(v, n - 1)
        v = np.where(inter, v, np.clip(v, c * m, last[c]))
        keep = u != v
        u, v = u[keep], v[keep]
        key = np.minimum(u, v).astype(np.int64) * n + np.maximum(u, v)
        have = np.unique(np.concatenate([have, key]))
    if have.size > target:
        have = np.sort(rng.choice(have, size=target, replace=False))
    u, v = have // n, have % n
    w = (1.0 - rng.random(have.size)).astype(np.float32)
    u, v = _relabel(n, u, v, rng)
    return _build_csr(n, u, v, w, {"generator": "powerlaw", "communities": n_comm,
                                   "tail": tail, "mix": mix, "edges": int(target)})


# ---------------------------------------------------------------- c3/c5: Gaussian kernel
def gaussian_points(n: int, dim: int, n_comp: int, rng: np.random.Generator,
                    mean_std: float = 3.0, sigma_pairs: int = 1_000_000):
    """Mixture points (means ~ N(0, mean_std^2 I), unit covariance, equal
    weights) and sigma = median pairwise distance over `sigma_pairs` seeded
    random pairs i != j (reading Z23)."""
    comp = rng.integers(0, n_comp, n)
    means = rng.normal(0.0, mean_std, size=(n_comp, dim))
    X = means[comp] + rng.normal(0.0, 1.0, size=(n, dim))
    i = rng.integers(0, n, sigma_pairs)
    j = rng.integers(0, n, sigma_pairs)
    keep = i != j
    d = np.sqrt(((X[i[keep]] - X[j[keep]]) ** 2).sum(axis=1))
    return X, float(np.median(d))


def gaussian_kernel_rows(X: np.ndarray, sigma: float, r0: int, r1: int,
                         col_block: int = 4096) -> np.ndarray:
    """Rows r0..r1-1 of A_ij = exp(-||x_i - x_j||^2 / sigma^2) as fp32.

    The squared distance is summed over dimensions in a fixed order from exact
    differences, so A_ij and A_ji are bitwise identical (exact symmetry), and
    any row block reproduces the same bits (the oracle regenerates rows).
    """
    n = X.shape[0]
    Xb = X[r0:r1]
    XT = np.ascontiguousarray(X.T)
    out = np.empty((r1 - r0, n), dtype=np.float32)
    for c0 in range(0, n, col_block):
        c1 = min(n, c0 + col_block)
        d2 = np.zeros((r1 - r0, c1 - c0))
        tmp = np.empty_like(d2)
        for d in range(X.shape[1]):
            np.subtract(Xb[:, d, None], XT[d, None, c0:c1], out=tmp)
            np.multiply(tmp, tmp, out=tmp)
            d2 += tmp
        d2 *= -1.0 / (sigma * sigma)
        np.exp(d2, out=d2)
        out[:, c0:c1] = d2
    return out


def gaussian_kernel_dense(X: np.ndarray, sigma: float, out: np.ndarray | None = None,
                          block: int = 64, threads: int | None = None) -> np.ndarray:
    n = X.shape[0]
    if out is None:
        out = np.empty((n, n), dtype=np.float32)
    threads = threads or min(32, os.cpu_count() or 1)

    def work(r0):
        r1 = min(n, r0 + block)
        out[r0:r1] = gaussian_kernel_rows(X, sigma, r0, r1)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(0, n, block)))
    return out


# ---------------------------------------------------------------- init and alpha
def alpha_of(A) -> float:
    """alpha = max(A) over all entries (reading Z14); exact in fp32."""
    if isinstance(A, CsrMatrix):
        return float(max(0.0, float(A.val.max()))) if A.nnz else 0.0
    return float(A.max())


def mean_entry(A) -> float:
    """zeta = sum_ij A_ij / n^2, zeros included (reading Z15)."""
    if isinstance(A, CsrMatrix):
        return float(A.val.astype(np.float64).sum()) / (A.n * A.n)
    n = A.shape[0]
    tot = 0.0
    for r0 in range(0, n, 4096):
        tot += float(A[r0:r0 + 4096].astype(np.float64).sum())
    return tot / (n * n)


def init_factor(n: int, k: int, zeta: float, rng: np.random.Generator) -> np.ndarray:
    """H0 = U[0,1) * 2 sqrt(zeta / k), fp32."""
    return (rng.random((n, k)) * (2.0 * math.sqrt(max(zeta, 0.0) / k))).astype(np.float32)


def random_factor(n: int, k: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """A generic seeded nonnegative fp32 n x k factor for unit-level parity tests."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, n, k])))
    return (rng.random((n, k)) * scale).astype(np.float32)


# ---------------------------------------------------------------- top level
def _cache_dir(name: str, seed: int, noise: bool, n: int):
    """Directory caching a large generated input (SYMNMF_INPUT_CACHE, default /tmp/symnmf_inputs;
    "off" disables), keyed by the recipe (config, seed, noise, n) and this file's bytes, so a cached
    input is the same bits a fresh draw gives.  Generation is outside every timed region; the
    cache only saves minutes when several runs of one session use c3/c4."""
    root = os.environ.get("SYMNMF_INPUT_CACHE", "/tmp/symnmf_inputs")
    if root == "off" or name not in ("c3", "c4") or n < 100_000 and name == "c4":
        return None
    import hashlib
    h = hashlib.sha1(open(__file__, "rb").read()).hexdigest()[:12]
    return os.path.join(root, f"{name}_s{seed}_n{n}_{int(noise)}_{h}")


def _cache_load(d):
    try:
        if d is None or not os.path.exists(os.path.join(d, "done")):
            return None
        z = {f[:-4]: np.load(os.path.join(d, f)) for f in os.listdir(d) if f.endswith(".npy")}
        if "rowptr" in z:
            return CsrMatrix(int(z["n"]), z["rowptr"], z["colidx"], z["val"]), z
        return z["A"], z
    except Exception:
        return None


def _cache_save(d, A, extra):
    try:
        os.makedirs(d, exist_ok=True)
        if isinstance(A, CsrMatrix):
            for k_, v in (("rowptr", A.rowptr), ("colidx", A.colidx), ("val", A.val), ("n", np.array(A.n))):
                np.save(os.path.join(d, k_ + ".npy"), v)
        else:
            np.save(os.path.join(d, "A.npy"), A)
        for k_ in ("points", "sigma"):
            if k_ in extra:
                np.save(os.path.join(d, k_ + ".npy"), np.asarray(extra[k_]))
        open(os.path.join(d, "done"), "w").close()
    except Exception:
        pass


def make_input(name: str, seed: int | None = None, noise: bool = True, n_override: int | None = None):
    """Generate config `name`.  Returns dict(cfg, A, H0, alpha, zeta, extra).

    `n_override` shrinks a config (same recipe, fewer rows) for CPU tests.
    """
    cfg = CONFIGS[name]
    seed = cfg.seed if seed is None else seed
    n = n_override or cfg.n
    drng, irng = _streams(seed)
    extra = {}
    cdir = _cache_dir(name, seed, noise, n)
    hit = _cache_load(cdir)
    if hit is not None:
        A, z = hit
        if "points" in z:
            extra.update(points=z["points"], sigma=float(z["sigma"]))
        zeta = mean_entry(A)
        H0 = init_factor(n, cfg.k, zeta, irng)
        return {"cfg": cfg, "n": n, "A": A, "H0": H0, "alpha": alpha_of(A), "zeta": zeta,
                "seed": seed, "extra": extra}
    if name == "c1":
        A, H0p = planted_dense(n, cfg.k, 0.01 if noise else 0.0, drng)
        extra["H0_planted"] = H0p
    elif name == "c2":
        A = sbm_csr(n, 16, 18.0, 2.0, drng)
    elif name == "c4":
        A = powerlaw_csr(n, 32, 50.0, 1.5, 0.1, drng)
    elif name in ("c3", "c5"):
        dim, comp = (64, 32) if name == "c3" else (128, 64)
        X, sigma = gaussian_points(n, dim, comp, drng)
        A = gaussian_kernel_dense(X, sigma)
        extra.update(points=X, sigma=sigma)
    else:
        raise KeyError(name)
    if cdir is not None:
        _cache_save(cdir, A, extra)
    zeta = mean_entry(A)
    H0 = init_factor(n, cfg.k, zeta, irng)
    return {"cfg": cfg, "n": n, "A": A, "H0": H0, "alpha": alpha_of(A), "zeta": zeta,
            "seed": seed, "extra": extra}
