"""CPU oracle for the AJM hot path -- TEST INFRASTRUCTURE, not product code.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may
import this package.  The product path (paper_2407_03272_b200) never imports it and shares no code
with it.  The arithmetic lives in plain C (ajm_oracle.c, FP64, -ffp-contract=off); this module only
builds it with gcc and marshals numpy arrays through ctypes.

Each function cites the passage it follows (PAPER.md = P, SPEC.md = S, readings R#):
  spmv            Q x, ascending-column row sums                       (P:463 Q y^t)
  build_jdiag     eq-J-diag  J_kk = Q_kk + sum_{j!=k}|Q_kj|
  build_jblock    eq-J-blkdiag J^{ii} = Q^{ii} + sum_{j!=i}||Q^{ij}||_2 I  (R23)
  diag            D = diag(Q)
  alpha_next      alpha_{t+1} = (1 + sqrt(1 + 4 alpha_t^2))/2
  objective       f(x) = 1/2<x,Qx> - <b,x>
  rel_residual    ||b - Qx|| / ||b||
  solve           Alg. 3, s = 1, literal two-SpMV form                 (R5-R10, R19)
  spectrum        extreme eigenvalues of D^{-1} Q and omega_opt = 2/(lmin + lmax)

Pins: tests/test_oracle_pins.py ties every function above to something other than itself (SPEC
worked values, dense Cholesky / pseudo-inverse solves, Thm 2.3 / Lemma 2.2 / Lemma 2.4 / Thm 2.5,
the restart-count bound, the alpha identities, the Jacobi / weighted-Jacobi reductions and the
§4.1 closed forms).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ajm_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libajm_oracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        lib.oracle_spmv.argtypes = [I64, P, P, P, P, P]
        lib.oracle_build_jdiag.argtypes = [I64, P, P, P, P]
        lib.oracle_build_jdiag.restype = ctypes.c_int
        lib.oracle_diag.argtypes = [I64, P, P, P, P]
        lib.oracle_alpha_next.argtypes = [ctypes.c_double]
        lib.oracle_alpha_next.restype = ctypes.c_double
        lib.oracle_objective.argtypes = [I64, P, P, P, P, P]
        lib.oracle_objective.restype = ctypes.c_double
        lib.oracle_rel_residual.argtypes = [I64, P, P, P, P, P]
        lib.oracle_rel_residual.restype = ctypes.c_double
        lib.oracle_dot.argtypes = [I64, P, P]
        lib.oracle_dot.restype = ctypes.c_double
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_get_threads.restype = ctypes.c_int
        lib.oracle_ajm_solve.argtypes = [I64, P, P, P, P, P, P, ctypes.c_double, I64, ctypes.c_int,
                                         ctypes.c_int, I64, ctypes.c_int, P, I64, P, P, P, P, P, P,
                                         P, P, P, I64, P]
        lib.oracle_ajm_solve.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _csr(Q):
    rp = np.ascontiguousarray(Q.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(Q.col, dtype=np.int32)
    v = np.ascontiguousarray(Q.val, dtype=np.float64)
    return rp, ci, v


def _vec(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def set_threads(nt: int) -> None:
    _load().oracle_set_threads(int(nt))


def get_threads() -> int:
    return int(_load().oracle_get_threads())


def spmv(Q, x) -> np.ndarray:
    rp, ci, v = _csr(Q)
    x = _vec(x)
    y = np.empty(Q.n)
    _load().oracle_spmv(Q.n, _p(rp), _p(ci), _p(v), _p(x), _p(y))
    return y


class OracleError(ValueError):
    pass


def build_jdiag(Q) -> np.ndarray:
    rp, ci, v = _csr(Q)
    J = np.empty(Q.n)
    err = _load().oracle_build_jdiag(Q.n, _p(rp), _p(ci), _p(v), _p(J))
    if err:
        raise OracleError({1: "negative diagonal", 2: "zero row (J_kk = 0)", 3: "non-finite value"}[err])
    return J


def build_jblock(Q, bs: int, batch: int = 1 << 16) -> np.ndarray:
    """eq-J-blkdiag: J = diag(J^{1,1}, ..., J^{s,s}) over contiguous row blocks of bs
    rows (block i = rows [i*bs, min((i+1)*bs, n)), the last one ragged -- DESIGN.md R23), with
        J^{ii} = Q^{ii} + (sum_{j != i} ||Q^{ij}||_2) I.
    ||Q^{ij}||_2 is the largest singular value of the dense off-diagonal block (numpy's LAPACK
    SVD); the shifts are summed in ascending j.  Returns the dense blocks, shape (s, bs, bs); the
    ragged last block is padded with the identity (which leaves J^{-1} on its rows unchanged)."""
    n = int(Q.n)
    bs = int(bs)
    if bs < 1:
        raise OracleError("block size must be >= 1")
    nblk = (n + bs - 1) // bs
    rp = np.asarray(Q.row_ptr, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    cols = np.asarray(Q.col, dtype=np.int64)
    vals = np.asarray(Q.val, dtype=np.float64)
    if not np.all(np.isfinite(vals)):
        raise OracleError("non-finite value")
    bi, bj = rows // bs, cols // bs
    J = np.zeros((nblk, bs, bs))
    on = bi == bj
    J[bi[on], rows[on] % bs, cols[on] % bs] = vals[on]       # Q^{ii}
    off = ~on
    key = bi[off] * nblk + bj[off]                           # sorted by (i, j): CSR order
    order = np.argsort(key, kind="stable")
    key, r_off, c_off, v_off = key[order], rows[off][order], cols[off][order], vals[off][order]
    uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
    norms = np.empty(len(uniq))
    for s0 in range(0, len(uniq), batch):                   # ||Q^{ij}||_2, batched SVDs
        s1 = min(s0 + batch, len(uniq))
        lo, hi = first[s0], (first[s1] if s1 < len(uniq) else len(key))
        B = np.zeros((s1 - s0, bs, bs))
        B[inv[lo:hi] - s0, r_off[lo:hi] % bs, c_off[lo:hi] % bs] = v_off[lo:hi]
        norms[s0:s1] = np.linalg.svd(B, compute_uv=False)[:, 0] if s1 > s0 else 0.0
    shift = np.zeros(nblk)
    for blk, nv in zip(uniq // nblk, norms):                 # ascending j within each i
        shift[blk] += nv
    idx = np.arange(bs)
    J[:, idx, idx] += shift[:, None]
    m = n - (nblk - 1) * bs                                  # ragged last block: identity pad
    for k in range(m, bs):
        J[nblk - 1, k, :] = 0.0
        J[nblk - 1, :, k] = 0.0
        J[nblk - 1, k, k] = 1.0
    return J


def jblock_factor(J: np.ndarray) -> np.ndarray:
    """Per-block lower Cholesky factors (LAPACK) of an eq-J-blkdiag J; an SPD failure raises
    (impossible for SPSD Q with exact norms)."""
    try:
        return np.ascontiguousarray(np.linalg.cholesky(J))
    except np.linalg.LinAlgError as e:
        raise OracleError(f"J block not SPD: {e}")


def diag(Q) -> np.ndarray:
    rp, ci, v = _csr(Q)
    d = np.empty(Q.n)
    _load().oracle_diag(Q.n, _p(rp), _p(ci), _p(v), _p(d))
    return d


def alpha_next(a: float) -> float:
    return float(_load().oracle_alpha_next(float(a)))


def objective(Q, b, x) -> float:
    rp, ci, v = _csr(Q)
    return float(_load().oracle_objective(Q.n, _p(rp), _p(ci), _p(v), _p(_vec(b)), _p(_vec(x))))


def rel_residual(Q, b, x) -> float:
    rp, ci, v = _csr(Q)
    r = float(_load().oracle_rel_residual(Q.n, _p(rp), _p(ci), _p(v), _p(_vec(b)), _p(_vec(x))))
    if np.isnan(r):
        raise OracleError("||b|| = 0: stopping rule undefined")
    return r


STATUS = {0: "converged", 1: "maxiter", 2: "diverged"}


@dataclasses.dataclass
class OracleResult:
    x: np.ndarray
    status: str
    iterations: int
    n_restarts: int
    x_is_prerestart: bool
    restart_iters: list
    res_hist: np.ndarray
    f_hist: np.ndarray
    d_hist: np.ndarray
    dabs_hist: np.ndarray
    xt_hist: np.ndarray | None
    alpha_hist: np.ndarray | None


def solve(Q, b, D=None, x0=None, tol=1e-6, maxit=1000, momentum=True, restart=True, k0=2,
          mirror=False, forced=None, record_iterates=False, dmode="jdiag",
          jblock: int | None = None) -> OracleResult:
    """Alg. 3.  D defaults to eq-J-diag; dmode='qdiag' uses diag(Q) (eq-jacobi);
    jblock=bs uses the block-diagonal J of eq-J-blkdiag with bs-row blocks (D is then ignored)."""
    rp, ci, v = _csr(Q)
    n = Q.n
    b = _vec(b)
    Lfac = None
    if jblock is not None:
        Lfac = jblock_factor(build_jblock(Q, jblock))
        D = np.ones(n)
    if D is None:
        D = build_jdiag(Q) if dmode == "jdiag" else diag(Q)
    D = _vec(D)
    x0a = None if x0 is None else _vec(x0)
    m1 = maxit + 1
    res_hist = np.zeros(m1)
    f_hist = np.zeros(m1)
    d_hist = np.zeros(m1)
    dabs_hist = np.zeros(m1)
    xt_hist = np.zeros(m1 * n) if record_iterates else None
    alpha_hist = np.zeros(m1) if record_iterates else None
    fa = None if forced is None else np.ascontiguousarray(forced, dtype=np.int8)
    cap = 4096
    rit = np.zeros(cap, dtype=np.int64)
    info = np.zeros(6, dtype=np.int64)
    x_out = np.empty(n)
    rc = _load().oracle_ajm_solve(n, _p(rp), _p(ci), _p(v), _p(b), _p(D), _p(x0a), float(tol),
                                  int(maxit), int(bool(momentum)), int(bool(restart)), int(k0),
                                  int(bool(mirror)), _p(fa), int(jblock or 0), _p(Lfac), _p(x_out), _p(res_hist), _p(f_hist),
                                  _p(d_hist), _p(dabs_hist), _p(xt_hist), _p(alpha_hist), _p(rit),
                                  cap, _p(info))
    if rc == -1:
        raise OracleError("invalid argument")
    if rc == -2:
        raise OracleError("||b|| = 0")
    if rc != 0:
        raise OracleError(f"oracle failure {rc}")
    it = int(info[1])
    k = it + 1
    return OracleResult(
        x=x_out, status=STATUS[int(info[0])], iterations=it, n_restarts=int(info[2]),
        x_is_prerestart=bool(info[3]), restart_iters=[int(r) for r in rit[: int(info[4])]],
        res_hist=res_hist[:k], f_hist=f_hist[:k], d_hist=d_hist[:k], dabs_hist=dabs_hist[:k],
        xt_hist=None if xt_hist is None else xt_hist.reshape(m1, n)[:k],
        alpha_hist=None if alpha_hist is None else alpha_hist[:k])


@dataclasses.dataclass
class OracleSpectrum:
    lambda_min: float
    lambda_max: float
    omega_opt: float
    method: str


def spectrum(Q, D=None, dmode: str = "qdiag", dense_max: int = 3000, tol: float = 1e-12) -> OracleSpectrum:
    """Extreme eigenvalues of D^{-1} Q for a positive diagonal metric D (default D = diag(Q), the
    Jacobi metric of P:54) and the optimal weighted-Jacobi weight
        omega_opt = 2 / (lambda_min(D^{-1} Q) + lambda_max(D^{-1} Q)).
    D^{-1} Q is similar to the symmetric D^{-1/2} Q D^{-1/2}, whose eigenvalues are
    computed by a library routine: LAPACK (numpy eigvalsh) on the dense matrix for n <= dense_max,
    else ARPACK (scipy eigsh, Lanczos with implicit restarts) for the two ends to `tol`."""
    if D is None:
        D = build_jdiag(Q) if dmode == "jdiag" else diag(Q)
    D = np.asarray(D, dtype=np.float64)
    if not np.all(D > 0):
        raise OracleError("the metric D must be positive")
    s = 1.0 / np.sqrt(D)
    n = int(Q.n)
    if n <= dense_max:
        A = np.zeros((n, n))
        rows = np.repeat(np.arange(n), np.diff(np.asarray(Q.row_ptr)))
        A[rows, np.asarray(Q.col)] = np.asarray(Q.val)
        A = s[:, None] * A * s[None, :]
        lam = np.linalg.eigvalsh(0.5 * (A + A.T))
        lmin, lmax, method = float(lam[0]), float(lam[-1]), "dense eigvalsh"
    else:
        import scipy.sparse as sp
        import scipy.sparse.linalg as spla
        A = sp.csr_matrix((np.asarray(Q.val), np.asarray(Q.col), np.asarray(Q.row_ptr)), shape=(n, n))
        A = sp.diags(s) @ A @ sp.diags(s)
        lmax = float(spla.eigsh(A, k=1, which="LA", tol=tol, return_eigenvectors=False)[0])
        # the low end by shift-and-invert around a point just below the spectrum (lmin >= 0: SPSD)
        lmin = float(spla.eigsh(A, k=1, sigma=-1e-3 * lmax, which="LM", tol=tol,
                                return_eigenvectors=False)[0])
        method = "ARPACK eigsh"
    return OracleSpectrum(lmin, lmax, 2.0 / (lmin + lmax), method)
