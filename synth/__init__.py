"""Seeded synthetic inputs for the AJM hot path (shared by the CUDA path's tests/bench and the oracle).

This module holds NO arithmetic of the method (no J, no iteration, no step): it only builds the
problem data Q (canonical CSR, both triangles stored), the planted solution x*, and b = Q x*
(the right-hand side the configs define; computed with scipy's library SpMV, which is input
preparation, not the method). Everything is deterministic in the seed (numpy PCG64).

Workloads (BASELINE.json ``configs``; recipes restated in DESIGN.md §3):
  1. poisson2d(64)                    2D 5-point Dirichlet Laplacian (diag 4, off -1)
  2. poisson3d(128)                   3D 7-point Dirichlet Laplacian (diag 6, off -1)
  3. er_laplacian(1_000_000, 8M)      weighted Erdos-Renyi Laplacian, singular SPSD
  4. chung_lu(4_000_000)              power-law (gamma 2.1) Laplacian + 1e-3 I
  5. aniso27(256)                     anisotropic 27-point stencil, SURVEY R20 reading
  plus the paper's §4.1 strictly diagonally dominant system sdd(n).

Stand-in note: the paper's SuiteSparse matrices are not in the
container; these synthetic matrices stand in for them (stencils for the PDE stiffness matrices,
ER/Chung-Lu Laplacians for the §4.2 graph Laplacians).
"""
from __future__ import annotations

import dataclasses
import os

import numpy as np

__all__ = [
    "CSR", "Problem", "poisson2d", "poisson3d", "aniso27", "er_laplacian", "chung_lu", "sdd",
    "random_spd", "random_laplacian", "diag_matrix", "from_dense", "to_dense", "make_problem",
    "CONFIGS", "config_problem", "random_vector",
]


@dataclasses.dataclass
class CSR:
    """Canonical CSR (row_ptr int64 [n+1], col int32 [nnz] strictly increasing per row, val f64)."""
    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.row_ptr), shape=(self.n, self.n))

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.row_ptr)


@dataclasses.dataclass
class Problem:
    name: str
    Q: CSR
    b: np.ndarray
    x_star: np.ndarray
    meta: dict


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def random_vector(n: int, seed: int, kind: str = "uniform") -> np.ndarray:
    """Seeded vector: 'uniform' U(-1,1) or 'normal_zero_mean' N(0,1) minus its mean."""
    g = _rng(seed)
    if kind == "uniform":
        return g.uniform(-1.0, 1.0, n)
    if kind == "normal_zero_mean":
        v = g.standard_normal(n)
        return v - v.mean()
    raise ValueError(kind)


# ----------------------------------------------------------------------------------------------
# structured grids
# ----------------------------------------------------------------------------------------------

def _stencil(m: int, dim: int, offsets, diag_mode: str, diag_value: float = 0.0,
             diag_shift: float = 0.0) -> CSR:
    """Dirichlet stencil on an m^dim grid, index i = x + m*y (+ m*m*z).

    offsets: list of (d tuple, coefficient) for the OFF-diagonal couplings (the centre is added
    here). diag_mode 'const' puts diag_value on every row (classical Dirichlet Laplacian);
    'absrow' puts sum_{j != i}|Q_ij| (ascending column order) + diag_shift.
    Columns are emitted in ascending order because offsets are sorted by linear offset.
    """
    n = m ** dim
    idx = np.arange(n, dtype=np.int64)
    coords = []
    rem = idx
    for _ in range(dim):
        coords.append((rem % m).astype(np.int32))
        rem = rem // m
    strides = [m ** a for a in range(dim)]
    full = [(tuple(0 for _ in range(dim)), None)] + list(offsets)
    full.sort(key=lambda dc: sum(d * s for d, s in zip(dc[0], strides)))

    def valid_mask(d):
        mask = np.ones(n, dtype=bool)
        for a in range(dim):
            if d[a] != 0:
                c = coords[a]
                mask &= (c + d[a] >= 0) & (c + d[a] < m)
        return mask

    counts = np.zeros(n, dtype=np.int64)
    masks = []
    for d, _ in full:
        mk = valid_mask(d)
        masks.append(mk)
        counts += mk
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    pos = row_ptr[:-1].copy()
    diag_pos = None
    absrow = np.zeros(n, dtype=np.float64)
    for (d, coef), mk in zip(full, masks):
        lin = sum(dd * s for dd, s in zip(d, strides))
        rows = idx[mk]
        p = pos[mk]
        col[p] = (rows + lin).astype(np.int32)
        if coef is None:
            diag_pos = (rows, p)
        else:
            val[p] = coef
            absrow[mk] += abs(coef)  # ascending column order: same offset sequence in every row
        pos[mk] += 1
        del rows, p
    rows, p = diag_pos
    if diag_mode == "const":
        val[p] = diag_value
    elif diag_mode == "absrow":
        val[p] = absrow + diag_shift
    else:
        raise ValueError(diag_mode)
    return CSR(n, row_ptr, col, val)


def poisson2d(m: int) -> CSR:
    """5-point Laplacian on an m x m interior grid, Dirichlet boundary: diag 4, neighbours -1."""
    offs = [((1, 0), -1.0), ((-1, 0), -1.0), ((0, 1), -1.0), ((0, -1), -1.0)]
    return _stencil(m, 2, offs, "const", 4.0)


def poisson3d(m: int) -> CSR:
    """7-point Laplacian on an m^3 grid, Dirichlet boundary: diag 6, neighbours -1."""
    offs = []
    for a in range(3):
        for s in (-1, 1):
            d = [0, 0, 0]
            d[a] = s
            offs.append((tuple(d), -1.0))
    return _stencil(m, 3, offs, "const", 6.0)


def aniso27(m: int, w=(1.0, 1.0, 1e-2), shift: float = 1e-6) -> CSR:
    """Anisotropic 27-point stencil (SURVEY R20 reading of BASELINE configs[4]).

    Q_{i,i+d} = -prod_{a: d_a != 0} w_a for d in {-1,0,1}^3 minus 0 (axis a of the grid index
    i = x + m*y + m^2*z has weight w[a]); Q_ii = sum_{j != i}|Q_ij| + shift.  Symmetric, strictly
    diagonally dominant, hence SPD.
    """
    offs = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                d = (dx, dy, dz)
                if d == (0, 0, 0):
                    continue
                c = 1.0
                for a in range(3):
                    if d[a] != 0:
                        c *= w[a]
                offs.append((d, -c))
    return _stencil(m, 3, offs, "absrow", diag_shift=shift)


# ----------------------------------------------------------------------------------------------
# graphs
# ----------------------------------------------------------------------------------------------

# Sorting kernels of the generators.  Large integer sorts / unique / searchsorted run through
# torch's multi-threaded CPU ops when torch is importable: for integer keys (and exact float
# comparisons in searchsorted) they return exactly numpy's results -- a stable sort's permutation
# and a sorted unique set are unique -- so the matrices are bitwise the same either way
# (tests/test_synth.py checks it); only the wall time of building configs 3-5 changes.
_FAST = os.environ.get("AJM_SYNTH_NUMPY") is None


def _torch():
    if not _FAST:
        return None
    try:
        import torch
        return torch
    except Exception:  # pragma: no cover
        return None


def _argsort_stable(key: np.ndarray) -> np.ndarray:
    torch = _torch()
    if torch is None or key.size < (1 << 20):
        return np.argsort(key, kind="stable")
    return torch.sort(torch.from_numpy(key), stable=True).indices.numpy()


def _unique(key: np.ndarray) -> np.ndarray:
    torch = _torch()
    if torch is None or key.size < (1 << 20):
        return np.unique(key)
    return torch.unique(torch.from_numpy(key), sorted=True).numpy()


def _searchsorted_right(cdf: np.ndarray, r: np.ndarray) -> np.ndarray:
    torch = _torch()
    if torch is None or r.size < (1 << 20):
        return np.searchsorted(cdf, r, side="right").astype(np.int64)
    return torch.searchsorted(torch.from_numpy(cdf), torch.from_numpy(r), right=True).numpy()


def _laplacian_from_edges(n: int, u: np.ndarray, v: np.ndarray, w: np.ndarray,
                          shift: float = 0.0) -> CSR:
    """L = Deg - W (+ shift*I) from an undirected simple edge list (u < v unique), CSR sorted."""
    rows = np.concatenate([u, v, np.arange(n, dtype=np.int64)])
    cols = np.concatenate([v, u, np.arange(n, dtype=np.int64)])
    deg = np.bincount(u, weights=w, minlength=n) + np.bincount(v, weights=w, minlength=n)
    vals = np.concatenate([-w, -w, deg + shift])
    key = rows * n + cols
    order = _argsort_stable(key)
    del key
    rows = rows[order]
    col = cols[order].astype(np.int32)
    val = vals[order]
    del order, cols, vals
    counts = np.bincount(rows, minlength=n)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return CSR(n, row_ptr, col, val)


def _dedupe_edges(n: int, u: np.ndarray, v: np.ndarray):
    keep = u != v
    u, v = u[keep], v[keep]
    a = np.minimum(u, v)
    bb = np.maximum(u, v)
    key = _unique(a.astype(np.int64) * n + bb)
    return key // n, key % n


def er_laplacian(n: int, m_edges: int, seed: int, wlo: float = 0.1, whi: float = 1.0) -> CSR:
    """Weighted G(n, m) Laplacian (singular SPSD).  m distinct edges uniformly at random, weights
    U(wlo, whi).  Any isolated vertex gets one extra edge to a uniformly drawn partner (SURVEY R2:
    no zero rows, since J_k = 0 is an error)."""
    g = _rng(seed)
    u = np.empty(0, np.int64)
    v = np.empty(0, np.int64)
    need = m_edges
    while True:
        du = g.integers(0, n, size=int(need * 1.05) + 16, dtype=np.int64)
        dv = g.integers(0, n, size=du.size, dtype=np.int64)
        u, v = _dedupe_edges(n, np.concatenate([u, du]), np.concatenate([v, dv]))
        if u.size >= m_edges:
            # keep a seeded random subset of exactly m edges
            sel = np.sort(g.choice(u.size, size=m_edges, replace=False))
            u, v = u[sel], v[sel]
            break
        need = m_edges - u.size
    deg = np.bincount(u, minlength=n) + np.bincount(v, minlength=n)
    iso = np.nonzero(deg == 0)[0]
    if iso.size:
        partner = g.integers(0, n - 1, size=iso.size, dtype=np.int64)
        partner = partner + (partner >= iso)  # avoid self loops
        u, v = _dedupe_edges(n, np.concatenate([u, iso]), np.concatenate([v, partner]))
    w = g.uniform(wlo, whi, u.size)
    return _laplacian_from_edges(n, u, v, w)


def chung_lu_weights(n: int, gamma: float = 2.1, mean_deg: float = 20.0,
                     w_max: float = 1e5) -> np.ndarray:
    """Expected degrees w_i = c (i + i0)^(-1/(gamma-1)) with mean mean_deg and max w_max
    (SURVEY R21); i0 found by bisection."""
    a = 1.0 / (gamma - 1.0)
    i = np.arange(n, dtype=np.float64)
    target = mean_deg / w_max

    def ratio(i0):  # mean(w)/max(w)
        return float(np.mean((i + i0) ** (-a)) / i0 ** (-a))

    lo, hi = 1e-6, float(n)
    for _ in range(200):
        mid = np.sqrt(lo * hi)
        if ratio(mid) < target:
            lo = mid
        else:
            hi = mid
    i0 = np.sqrt(lo * hi)
    w = (i + i0) ** (-a)
    return w * (mean_deg / w.mean())


def chung_lu(n: int, seed: int, gamma: float = 2.1, mean_deg: float = 20.0, w_max: float = 1e5,
             shift: float = 1e-3, wlo: float = 0.1, whi: float = 1.0) -> CSR:
    """Chung-Lu power-law graph Laplacian + shift*I (SPD).  m = sum(w)/2 endpoint pairs drawn
    independently proportional to w, self loops dropped, duplicates merged, weights U(wlo, whi)."""
    g = _rng(seed)
    wexp = chung_lu_weights(n, gamma, mean_deg, w_max)
    m = int(round(wexp.sum() / 2))
    cdf = np.cumsum(wexp)
    cdf /= cdf[-1]
    u = _searchsorted_right(cdf, g.random(m))
    v = _searchsorted_right(cdf, g.random(m))
    np.minimum(u, n - 1, out=u)
    np.minimum(v, n - 1, out=v)
    u, v = _dedupe_edges(n, u, v)
    w = g.uniform(wlo, whi, u.size)
    return _laplacian_from_edges(n, u, v, w, shift=shift)


# ----------------------------------------------------------------------------------------------
# small / paper matrices
# ----------------------------------------------------------------------------------------------

def from_dense(A: np.ndarray, drop_zeros: bool = True) -> CSR:
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    mask = (A != 0) if drop_zeros else np.ones_like(A, dtype=bool)
    counts = mask.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    r, c = np.nonzero(mask)
    return CSR(n, row_ptr, c.astype(np.int32), A[r, c].copy())


def to_dense(Q: CSR) -> np.ndarray:
    A = np.zeros((Q.n, Q.n))
    rows = np.repeat(np.arange(Q.n), np.diff(Q.row_ptr))
    A[rows, Q.col] = Q.val
    return A


def sdd(n: int) -> CSR:
    """PAPER.md:512-520 (§4.1): Q with n on the diagonal and -1 elsewhere (dense pattern)."""
    A = -np.ones((n, n))
    np.fill_diagonal(A, float(n))
    return from_dense(A)


def diag_matrix(d: np.ndarray) -> CSR:
    return from_dense(np.diag(np.asarray(d, dtype=np.float64)))


def random_spd(n: int, seed: int, density: float = 0.3, shift: float = 1e-1) -> CSR:
    """Tiny random sparse SPD: A = B B^T restricted to a symmetric pattern, then made diagonally
    positive definite by a Gershgorin-free route: A = M^T M + shift*I of a sparse M."""
    g = _rng(seed)
    M = g.standard_normal((n, n)) * (g.random((n, n)) < density)
    A = M.T @ M + shift * np.eye(n)
    A = 0.5 * (A + A.T)
    return from_dense(A)


def random_laplacian(n: int, seed: int, p: float = 0.3) -> CSR:
    """Tiny weighted connected graph Laplacian (singular SPSD): a random path keeps it connected."""
    g = _rng(seed)
    W = np.triu((g.random((n, n)) < p) * g.uniform(0.1, 1.0, (n, n)), 1)
    perm = g.permutation(n)
    for a, bb in zip(perm[:-1], perm[1:]):
        i, j = min(a, bb), max(a, bb)
        if W[i, j] == 0:
            W[i, j] = g.uniform(0.1, 1.0)
    W = W + W.T
    L = np.diag(W.sum(axis=1)) - W
    return from_dense(L)


def make_problem(name: str, Q: CSR, seed: int, xkind: str = "uniform", meta=None) -> Problem:
    x_star = random_vector(Q.n, seed, xkind)
    b = Q.scipy() @ x_star
    return Problem(name, Q, b, x_star, dict(meta or {}))


# ----------------------------------------------------------------------------------------------
# BASELINE.json configs; seed default = config index
# ----------------------------------------------------------------------------------------------

CONFIGS = {
    1: dict(name="poisson2d_64", desc="2D 5-pt Laplacian 64x64 Dirichlet"),
    2: dict(name="poisson3d_128", desc="3D 7-pt Laplacian 128^3 Dirichlet"),
    3: dict(name="er_1m_deg16", desc="weighted ER Laplacian n=1M mean degree 16 (singular)"),
    4: dict(name="chunglu_4m_deg20", desc="Chung-Lu gamma=2.1 n=4M mean degree 20 + 1e-3 I"),
    5: dict(name="aniso27_256", desc="anisotropic 27-pt 256^3, w=(1,1,1e-2), diag=absrow+1e-6"),
}


def config_problem(cfg: int, scale: float = 1.0, seed: int | None = None) -> Problem:
    """Build BASELINE config `cfg` (1..5).  scale < 1 shrinks it (grid edge or n) for the
    oracle-sized parity cases; scale = 1 is the full BASELINE size."""
    seed = cfg if seed is None else seed
    meta = dict(config=cfg, scale=scale, seed=seed, **CONFIGS[cfg])
    if cfg == 1:
        m = max(2, int(round(64 * scale)))
        return make_problem(CONFIGS[1]["name"], poisson2d(m), seed, meta=meta | {"m": m})
    if cfg == 2:
        m = max(2, int(round(128 * scale)))
        return make_problem(CONFIGS[2]["name"], poisson3d(m), seed, meta=meta | {"m": m})
    if cfg == 3:
        n = max(16, int(round(1_000_000 * scale)))
        Q = er_laplacian(n, 8 * n, seed)
        return make_problem(CONFIGS[3]["name"], Q, seed + 1000, "normal_zero_mean",
                            meta=meta | {"n": n})
    if cfg == 4:
        n = max(64, int(round(4_000_000 * scale)))
        wmax = 1e5 * (n / 4_000_000) ** (1.0 / 1.1)  # keep the power-law head proportional
        Q = chung_lu(n, seed, w_max=max(wmax, 40.0))
        return make_problem(CONFIGS[4]["name"], Q, seed + 1000, meta=meta | {"n": n})
    if cfg == 5:
        m = max(3, int(round(256 * scale)))
        return make_problem(CONFIGS[5]["name"], aniso27(m), seed, meta=meta | {"m": m})
    raise ValueError(cfg)
