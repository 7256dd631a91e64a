"""paper_2407_03272_b200 -- B200-native accelerated Jacobi-type method (arXiv 2407.03272, Alg. 3).

Thin ctypes binding of libajm.so (C ABI in include/ajm.h).  Argument marshalling only: every step
of the method runs in the library's sm_100a kernels.  There is no CPU fallback -- if libajm.so
is missing, or no CUDA device is present when a solver is created, the calls raise.

Names follow the ABI: ``ajm_create`` / ``ajm_solve`` / ``ajm_destroy`` (+ ``Solver``, a handle
wrapper).  Arrays may be numpy arrays (host) or torch tensors (host or CUDA); PyTorch is only
used for device memory and streams.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np

__all__ = ["AjmError", "Result", "Solver", "Spectrum", "ShardGroup", "ShardSolver", "ajm_create", "ajm_solve",
           "ajm_destroy", "ajm_partition_rows", "ajm_shard_plan", "shard_rows", "lib", "LIB_PATH",
           "STATUS_NAMES", "TERM_NAMES", "D_MODES", "model_bytes_per_iter"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libajm.so")
if os.environ.get("AJM_LIB_OVERRIDE"):  # A/B experiments against another build of the same ABI
    LIB_PATH = os.environ["AJM_LIB_OVERRIDE"]

STATUS_NAMES = {0: "AJM_OK", 1: "AJM_ERR_INVALID_ARG", 2: "AJM_ERR_CSR_INVALID",
                3: "AJM_ERR_NOT_SYMMETRIC", 4: "AJM_ERR_NONFINITE", 5: "AJM_ERR_NEGATIVE_DIAG",
                6: "AJM_ERR_ZERO_DIAG", 7: "AJM_ERR_ZERO_RHS", 8: "AJM_ERR_CUDA", 9: "AJM_ERR_OOM",
                10: "AJM_ERR_UNSUPPORTED"}
TERM_NAMES = {0: "converged", 1: "maxiter", 2: "diverged"}
D_MODES = {"jdiag": 0, "user": 1, "qdiag": 2, "jblock": 3}
AJM_VALIDATE_SYMMETRY = 0x1
AJM_LOOP_HOST = 0x10
AJM_INT32_COLUMNS = 0x10000
AJM_GLOBAL_TABLES = 0x20000
AJM_SEGMENTS_STATIC = 0x40000
AJM_SEGMENTS_DYNAMIC = 0x80000
AJM_DEBUG_POISON = 0x100000
AJM_SHARD_COLOCATED = 0x200000
AJM_VALUE_STREAM = 0x400000
AJM_NO_BAND_STAGING = 0x800000
AJM_MAX_RANKS = 8
AJM_SHARD_BLOB_BYTES = 1024
ABI_VERSION = 5


def AJM_JBLOCK_SIZE(bs: int) -> int:
    """Create-flag bits carrying the eq-J-blkdiag block size (include/ajm.h)."""
    return (int(bs) & 0xFF) << 8

# every symbol include/ajm.h declares (tests check the .so exports all of them)
ABI_SYMBOLS = ["ajm_create", "ajm_solve", "ajm_get_trace", "ajm_get_diag", "ajm_get_jblock",
               "ajm_estimate_spectrum", "ajm_get_info", "ajm_destroy", "ajm_last_error",
               "ajm_abi_version", "ajm_partition_rows", "ajm_shard_plan", "ajm_shard_create",
               "ajm_shard_export", "ajm_shard_connect", "ajm_group_solve"]


class AjmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.status_name = STATUS_NAMES.get(status, str(status))


class ajm_policy_t(ctypes.Structure):
    _fields_ = [("momentum", ctypes.c_int32), ("restart", ctypes.c_int32), ("k0", ctypes.c_int64)]


class ajm_result_t(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("n_restarts", ctypes.c_int32),
                ("iterations", ctypes.c_int64), ("rel_residual", ctypes.c_double),
                ("f", ctypes.c_double), ("x_is_prerestart", ctypes.c_int32),
                ("restarts_logged", ctypes.c_int32)]


class ajm_info_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("units", ctypes.c_int64),
                ("long_rows", ctypes.c_int64), ("grid", ctypes.c_int32), ("block", ctypes.c_int32),
                ("sm_count", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32),
                ("model_bytes_per_iter", ctypes.c_double), ("last_loop_ms", ctypes.c_double),
                ("last_passes", ctypes.c_int64), ("last_launches", ctypes.c_int64),
                ("sell_rows", ctypes.c_int64), ("seg_rows", ctypes.c_int64),
                ("split_rows", ctypes.c_int64), ("sell_elems", ctypes.c_int64),
                ("sigma", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("l2_window_bytes", ctypes.c_int64), ("l2_hit_ratio", ctypes.c_double),
                ("mode", ctypes.c_int32), ("l2_mode", ctypes.c_int32),
                ("launches_per_solve", ctypes.c_int32), ("col_bytes", ctypes.c_int32),
                ("seg_nnz", ctypes.c_int64), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("halo", ctypes.c_int64), ("send", ctypes.c_int64), ("group_rows", ctypes.c_int64),
                ("val_bytes", ctypes.c_int32), ("band_staged", ctypes.c_int32)]


class ajm_spectrum_t(ctypes.Structure):
    _fields_ = [("lambda_min", ctypes.c_double), ("lambda_max", ctypes.c_double),
                ("err_min", ctypes.c_double), ("err_max", ctypes.c_double),
                ("omega_opt", ctypes.c_double), ("steps", ctypes.c_int64),
                ("converged", ctypes.c_int32), ("breakdown", ctypes.c_int32)]


@dataclasses.dataclass
class Spectrum:
    """Extreme eigenvalues of D^{-1} Q (ajm_estimate_spectrum) and omega_opt = 2/(lmin + lmax)."""
    lambda_min: float
    lambda_max: float
    err_min: float
    err_max: float
    omega_opt: float
    steps: int
    converged: bool
    breakdown: bool
    alpha: np.ndarray
    beta: np.ndarray


_lib = None


def lib():
    """Load libajm.so (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() or "
                              "python paper_2407_03272_b200/build.py")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.ajm_create.argtypes = [ctypes.POINTER(P), I64, I64, P, P, P, P, ctypes.c_int32, P,
                                 ctypes.c_uint32, P]
        L.ajm_create.restype = ctypes.c_int
        L.ajm_solve.argtypes = [P, P, ctypes.c_double, I64, ajm_policy_t, P,
                                ctypes.POINTER(ajm_result_t), P, P, P, I64, P]
        L.ajm_solve.restype = ctypes.c_int
        L.ajm_get_trace.argtypes = [P, ctypes.c_int32, P, I64]
        L.ajm_get_trace.restype = ctypes.c_int
        L.ajm_get_diag.argtypes = [P, P]
        L.ajm_get_diag.restype = ctypes.c_int
        if hasattr(L, "ajm_get_jblock"):  # (AJM_LIB_OVERRIDE A/B builds may predate it)
            L.ajm_get_jblock.argtypes = [P, P]
            L.ajm_get_jblock.restype = ctypes.c_int
        if hasattr(L, "ajm_estimate_spectrum"):
            L.ajm_estimate_spectrum.argtypes = [P, P, ctypes.c_uint64, I64, ctypes.c_double,
                                                ctypes.POINTER(ajm_spectrum_t), P, P, P]
            L.ajm_estimate_spectrum.restype = ctypes.c_int
        L.ajm_get_info.argtypes = [P, ctypes.POINTER(ajm_info_t)]
        L.ajm_get_info.restype = ctypes.c_int
        L.ajm_destroy.argtypes = [P]
        L.ajm_destroy.restype = ctypes.c_int
        L.ajm_last_error.argtypes = [P]
        L.ajm_last_error.restype = ctypes.c_char_p
        L.ajm_abi_version.restype = ctypes.c_int32
        if hasattr(L, "ajm_shard_create"):
            L.ajm_partition_rows.argtypes = [I64, P, ctypes.c_int32, P]
            L.ajm_partition_rows.restype = ctypes.c_int
            L.ajm_shard_plan.argtypes = [ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, P, P]
            L.ajm_shard_plan.restype = ctypes.c_int
            L.ajm_shard_create.argtypes = [ctypes.POINTER(P), ctypes.c_int32, ctypes.c_int32, P, I64, P, P, P,
                                           P, ctypes.c_int32, P, ctypes.c_uint32, P]
            L.ajm_shard_create.restype = ctypes.c_int
            L.ajm_shard_export.argtypes = [P, P]
            L.ajm_shard_export.restype = ctypes.c_int
            L.ajm_shard_connect.argtypes = [P, P]
            L.ajm_shard_connect.restype = ctypes.c_int
            L.ajm_group_solve.argtypes = [P, ctypes.c_int32, P, ctypes.c_double, I64, ajm_policy_t, P,
                                          ctypes.POINTER(ajm_result_t), P, P, P, I64, P]
            L.ajm_group_solve.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a, dtype, output=False):
    """(pointer, keepalive) of a numpy array or torch tensor with the given numpy dtype.

    Inputs are converted (a contiguous copy of the right dtype) when needed.  Outputs are written
    by the library in place, so a converted temporary would silently drop the result: an output
    of the wrong dtype, or not contiguous, raises instead."""
    if a is None:
        return None, None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            tdt = {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[dtype]
            if a.dtype != tdt or not a.is_contiguous():
                if output:
                    raise TypeError(f"output tensor must be a contiguous {tdt} tensor "
                                    f"(got {a.dtype}, contiguous={a.is_contiguous()})")
                a = a.to(tdt).contiguous()
            return ctypes.c_void_p(a.data_ptr()), a
    except ImportError:  # pragma: no cover
        pass
    if output:
        if not (isinstance(a, np.ndarray) and a.dtype == np.dtype(dtype) and a.flags.c_contiguous
                and a.flags.writeable):
            raise TypeError(f"output array must be a writeable C-contiguous numpy {np.dtype(dtype)} array")
        return a.ctypes.data_as(ctypes.c_void_p), a
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data_as(ctypes.c_void_p), arr


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _check(st: int, handle=None):
    if st != 0:
        msg = lib().ajm_last_error(handle)
        raise AjmError(st, msg.decode() if msg else "")


def model_bytes_per_iter(n: int, nnz: int) -> float:
    """Algorithmic bytes of one fused pass: nnz*12 + 7 vectors * n * 8 + int32 row_ptr
    (DESIGN.md §4)."""
    return 12.0 * nnz + 56.0 * n + 4.0 * (n + 1)


def ajm_create(n, nnz, row_ptr, col_idx, vals, b, dmode="jdiag", d=None, flags=0, stream=None):
    """Marshal to ajm_create; returns the opaque handle (int)."""
    keep = []
    ptrs = []
    for a, dt in ((row_ptr, np.int64), (col_idx, np.int32), (vals, np.float64), (b, np.float64),
                  (d, np.float64)):
        p, k = _ptr(a, dt)
        ptrs.append(p)
        keep.append(k)
    h = ctypes.c_void_p()
    dm = D_MODES[dmode] if isinstance(dmode, str) else int(dmode)
    st = lib().ajm_create(ctypes.byref(h), int(n), int(nnz), ptrs[0], ptrs[1], ptrs[2], ptrs[3],
                          dm, ptrs[4], int(flags), _stream(stream))
    _check(st, None)
    return h.value


def ajm_solve(handle, x0, tol, maxit, momentum=True, restart=True, k0=2, x_out=None,
              res_hist=None, f_hist=None, restart_iters=None, stream=None):
    """Marshal to ajm_solve; returns the ajm_result_t."""
    p0, k_0 = _ptr(x0, np.float64)
    px, k_x = _ptr(x_out, np.float64, output=True)
    pr, k_r = _ptr(res_hist, np.float64, output=True)
    pf, k_f = _ptr(f_hist, np.float64, output=True)
    pri, k_ri = _ptr(restart_iters, np.int64, output=True)
    cap = 0 if restart_iters is None else len(restart_iters)
    res = ajm_result_t()
    pol = ajm_policy_t(int(bool(momentum)), int(bool(restart)), int(k0))
    st = lib().ajm_solve(ctypes.c_void_p(handle), p0, float(tol), int(maxit), pol, px,
                         ctypes.byref(res), pr, pf, pri, cap, _stream(stream))
    _check(st, ctypes.c_void_p(handle))
    return res


def ajm_destroy(handle):
    if handle:
        _check(lib().ajm_destroy(ctypes.c_void_p(handle)))


@dataclasses.dataclass
class Result:
    x: object
    status: str
    iterations: int
    rel_residual: float
    f: float
    n_restarts: int
    x_is_prerestart: bool
    restart_iters: list
    res_hist: np.ndarray | None
    f_hist: np.ndarray | None


class Solver:
    """Handle wrapper: ``Solver(Q_csr_arrays, b, dmode, d).solve(x0, tol, maxit, policy)``.

    row_ptr/col/val/b/d may be numpy arrays (copied host->device by the library) or torch tensors
    (device arrays are copied device->device).  The solver owns its device copy afterwards."""

    def __init__(self, n, row_ptr, col, val, b, dmode="jdiag", d=None, validate_symmetry=False,
                 loop="graph", stream=None, jblock=None, int32_columns=False, global_tables=False,
                 segments="auto", debug_poison=False, value_stream=False, band_staging=True):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2407_03272_b200 needs a CUDA device (no CPU fallback)")
        self.n = int(n)
        self.nnz = int(row_ptr[-1])
        flags = (AJM_VALIDATE_SYMMETRY if validate_symmetry else 0) | (AJM_LOOP_HOST if loop == "host" else 0)
        flags |= (AJM_INT32_COLUMNS if int32_columns else 0) | (AJM_GLOBAL_TABLES if global_tables else 0)
        flags |= {"auto": 0, "static": AJM_SEGMENTS_STATIC, "dynamic": AJM_SEGMENTS_DYNAMIC}[segments]
        flags |= AJM_DEBUG_POISON if debug_poison else 0
        flags |= AJM_VALUE_STREAM if value_stream else 0
        flags |= 0 if band_staging else AJM_NO_BAND_STAGING
        self.jblock = None
        if jblock is not None:  # eq-J-blkdiag with bs-row blocks (AJM_D_JBLOCK)
            dmode = "jblock"
            flags |= AJM_JBLOCK_SIZE(jblock)
            self.jblock = int(jblock)
        self._stream = stream
        self.handle = ajm_create(self.n, self.nnz, row_ptr, col, val, b, dmode, d, flags, stream)

    @classmethod
    def from_csr(cls, Q, b, **kw):
        return cls(Q.n, Q.row_ptr, Q.col, Q.val, b, **kw)

    def solve(self, x0=None, tol=1e-6, maxit=1000, momentum=True, restart=True, k0=2,
              x_out=None, history=True, restart_cap=64) -> Result:
        import torch
        if x_out is None:
            x_out = torch.empty(self.n, dtype=torch.float64, device="cuda")
        rh = np.empty(maxit + 1) if history else None
        fh = np.empty(maxit + 1) if history else None
        ri = np.zeros(restart_cap, dtype=np.int64)
        r = ajm_solve(self.handle, x0, tol, maxit, momentum, restart, k0, x_out, rh, fh, ri,
                      self._stream)
        k = r.iterations + 1
        return Result(x=x_out, status=TERM_NAMES[r.status], iterations=int(r.iterations),
                      rel_residual=r.rel_residual, f=r.f, n_restarts=int(r.n_restarts),
                      x_is_prerestart=bool(r.x_is_prerestart),
                      restart_iters=[int(v) for v in ri[: r.restarts_logged]],
                      res_hist=None if rh is None else rh[:k], f_hist=None if fh is None else fh[:k])

    def estimate_spectrum(self, v0=None, seed: int = 0, max_steps: int = 2000, tol: float = 1e-8) -> Spectrum:
        """Extreme eigenvalues of D^{-1} Q by Lanczos on the handle's own SpMV (ajm_estimate_spectrum)
        and omega_opt = 2 / (lambda_min + lambda_max), the optimal weighted-Jacobi weight for
        D = diag(Q) (create the solver with dmode="qdiag" for that metric)."""
        out = ajm_spectrum_t()
        a = np.zeros(max_steps)
        b = np.zeros(max_steps)
        p0, k0 = _ptr(v0, np.float64)
        _check(lib().ajm_estimate_spectrum(ctypes.c_void_p(self.handle), p0, int(seed), int(max_steps),
                                           float(tol), ctypes.byref(out), a.ctypes.data_as(ctypes.c_void_p),
                                           b.ctypes.data_as(ctypes.c_void_p), _stream(self._stream)),
               ctypes.c_void_p(self.handle))
        k = int(out.steps)
        return Spectrum(out.lambda_min, out.lambda_max, out.err_min, out.err_max, out.omega_opt, k,
                        bool(out.converged), bool(out.breakdown), a[:k].copy(), b[:k].copy())

    def trace(self, which: str, count: int) -> np.ndarray:
        out = np.empty(count)
        w = {"res": 0, "f": 1, "d": 2, "dabs": 3}[which]
        _check(lib().ajm_get_trace(ctypes.c_void_p(self.handle), w, out.ctypes.data_as(ctypes.c_void_p),
                                   int(count)), ctypes.c_void_p(self.handle))
        return out

    def diag(self) -> np.ndarray:
        out = np.empty(self.n)
        _check(lib().ajm_get_diag(ctypes.c_void_p(self.handle), out.ctypes.data_as(ctypes.c_void_p)),
               ctypes.c_void_p(self.handle))
        return out

    def jblocks(self) -> np.ndarray:
        """The blocks J^{ii} of eq-J-blkdiag built by the library, shape (s, bs, bs)."""
        if not self.jblock:
            raise ValueError("solver was not created with jblock=bs")
        bs = self.jblock
        s = (self.n + bs - 1) // bs
        out = np.empty(s * bs * bs)
        _check(lib().ajm_get_jblock(ctypes.c_void_p(self.handle), out.ctypes.data_as(ctypes.c_void_p)),
               ctypes.c_void_p(self.handle))
        return out.reshape(s, bs, bs)

    def info(self) -> dict:
        inf = ajm_info_t()
        _check(lib().ajm_get_info(ctypes.c_void_p(self.handle), ctypes.byref(inf)),
               ctypes.c_void_p(self.handle))
        return {f: getattr(inf, f) for f, _ in ajm_info_t._fields_}

    def close(self):
        if getattr(self, "handle", None):
            ajm_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- row-block sharded solve (NEXT-2; include/ajm.h "Row-block sharded solve") ----

def ajm_partition_rows(row_ptr, nranks: int) -> np.ndarray:
    """Contiguous row blocks balanced by the per-pass bytes (host only, no GPU): int64[nranks+1]."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    out = np.zeros(int(nranks) + 1, dtype=np.int64)
    _check(lib().ajm_partition_rows(len(rp) - 1, rp.ctypes.data_as(ctypes.c_void_p), int(nranks),
                                    out.ctypes.data_as(ctypes.c_void_p)))
    return out


def shard_rows(row_ptr, col, val, starts, rank: int):
    """The rows of block `rank` as (row_ptr rebased to 0, global columns, values): slicing only."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    r0, r1 = int(starts[rank]), int(starts[rank + 1])
    k0, k1 = int(rp[r0]), int(rp[r1])
    return rp[r0:r1 + 1] - k0, np.asarray(col)[k0:k1], np.asarray(val)[k0:k1]


def ajm_shard_plan(rank: int, nranks: int, starts, row_ptr_loc, col_glob) -> dict:
    """Host-only plan of one rank (no GPU): local columns, halo (global indices in local order), send
    lists grouped by destination rank, and the per-rank counts (include/ajm.h ajm_shard_plan)."""
    st = np.ascontiguousarray(starts, dtype=np.int64)
    rp = np.ascontiguousarray(row_ptr_loc, dtype=np.int64)
    cg = np.ascontiguousarray(col_glob, dtype=np.int32)
    R = int(nranks)
    counts = np.zeros(2 + 2 * R, dtype=np.int64)
    P = ctypes.c_void_p
    _check(lib().ajm_shard_plan(int(rank), R, st.ctypes.data_as(P), rp.ctypes.data_as(P), cg.ctypes.data_as(P),
                                None, None, None, counts.ctypes.data_as(P)))
    h_lo, h_hi = int(counts[0]), int(counts[1])
    col_loc = np.empty(len(cg), dtype=np.int32)
    halo = np.empty(h_lo + h_hi, dtype=np.int64)
    send = np.empty(int(counts[2 + R:].sum()), dtype=np.int64)
    _check(lib().ajm_shard_plan(int(rank), R, st.ctypes.data_as(P), rp.ctypes.data_as(P), cg.ctypes.data_as(P),
                                col_loc.ctypes.data_as(P), halo.ctypes.data_as(P), send.ctypes.data_as(P),
                                counts.ctypes.data_as(P)))
    return {"col_loc": col_loc, "halo_glob": halo, "send_rows": send, "h_lo": h_lo, "h_hi": h_hi,
            "halo_cnt": counts[2:2 + R].copy(), "send_cnt": counts[2 + R:].copy()}


def _shard_create(rank, nranks, starts, row_ptr_loc, col_glob, val, b_loc, dmode, d_loc, flags, stream):
    keep = []
    ptrs = []
    for a, dt in ((starts, np.int64), (row_ptr_loc, np.int64), (col_glob, np.int32), (val, np.float64),
                  (b_loc, np.float64), (d_loc, np.float64)):
        p, k = _ptr(a, dt)
        ptrs.append(p)
        keep.append(k)
    h = ctypes.c_void_p()
    dm = D_MODES[dmode] if isinstance(dmode, str) else int(dmode)
    nnz = int(np.asarray(row_ptr_loc[-1].cpu() if hasattr(row_ptr_loc, "cpu") else row_ptr_loc[-1]))
    _check(lib().ajm_shard_create(ctypes.byref(h), int(rank), int(nranks), ptrs[0], nnz, ptrs[1], ptrs[2],
                                  ptrs[3], ptrs[4], dm, ptrs[5], int(flags), _stream(stream)), None)
    return h.value


def _shard_export(handle) -> bytes:
    buf = ctypes.create_string_buffer(AJM_SHARD_BLOB_BYTES)
    _check(lib().ajm_shard_export(ctypes.c_void_p(handle), ctypes.cast(buf, ctypes.c_void_p)),
           ctypes.c_void_p(handle))
    return buf.raw


def _shard_connect(handle, blobs) -> None:
    joined = b"".join(blobs)
    assert len(joined) == AJM_SHARD_BLOB_BYTES * len(blobs)
    buf = ctypes.create_string_buffer(joined, len(joined))
    _check(lib().ajm_shard_connect(ctypes.c_void_p(handle), ctypes.cast(buf, ctypes.c_void_p)),
           ctypes.c_void_p(handle))


def _result(r, x_out, rh, fh, ri) -> Result:
    k = r.iterations + 1
    return Result(x=x_out, status=TERM_NAMES[r.status], iterations=int(r.iterations),
                  rel_residual=r.rel_residual, f=r.f, n_restarts=int(r.n_restarts),
                  x_is_prerestart=bool(r.x_is_prerestart),
                  restart_iters=[int(v) for v in ri[: r.restarts_logged]],
                  res_hist=None if rh is None else rh[:k], f_hist=None if fh is None else fh[:k])


class _ShardHandles:
    def _info(self, h) -> dict:
        inf = ajm_info_t()
        _check(lib().ajm_get_info(ctypes.c_void_p(h), ctypes.byref(inf)), ctypes.c_void_p(h))
        return {f: getattr(inf, f) for f, _ in ajm_info_t._fields_}

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardGroup(_ShardHandles):
    """All ranks of a row-block sharded solve on THIS device (AJM_SHARD_COLOCATED), solved as one
    cooperative launch (ajm_group_solve): the multi-GPU kernel and exchange with the peers being
    ordinary device pointers -- how the sharded path runs and is tested on a single GPU."""

    def __init__(self, n, row_ptr, col, val, b, nranks: int, starts=None, dmode="jdiag", d=None,
                 int32_columns=False, segments="auto", stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2407_03272_b200 needs a CUDA device (no CPU fallback)")
        self.n = int(n)
        self.nranks = int(nranks)
        self._stream = stream
        self.starts = ajm_partition_rows(row_ptr, nranks) if starts is None else np.asarray(starts, dtype=np.int64)
        flags = AJM_SHARD_COLOCATED | (AJM_INT32_COLUMNS if int32_columns else 0)
        flags |= {"auto": 0, "static": AJM_SEGMENTS_STATIC, "dynamic": AJM_SEGMENTS_DYNAMIC}[segments]
        self.handles = []
        bb = np.asarray(b, dtype=np.float64)
        dd = None if d is None else np.asarray(d, dtype=np.float64)

        def create_all(fl):
            for r in range(self.nranks):
                rp, cg, vv = shard_rows(row_ptr, col, val, self.starts, r)
                r0, r1 = int(self.starts[r]), int(self.starts[r + 1])
                self.handles.append(_shard_create(r, self.nranks, self.starts, rp, cg, vv, bb[r0:r1], dmode,
                                                  None if dd is None else dd[r0:r1], fl, stream))
        create_all(flags)
        # one launch runs every rank: they must share the column encoding (byte codes need every
        # rank's offsets to fit one table each -- a rank whose do not keeps int32 columns)
        if len({(self._info(h)["col_bytes"], self._info(h)["val_bytes"]) for h in self.handles}) > 1:
            self.close()
            create_all(flags | AJM_INT32_COLUMNS)
        blobs = [_shard_export(h) for h in self.handles]
        for h in self.handles:
            _shard_connect(h, blobs)

    @classmethod
    def from_csr(cls, Q, b, nranks, **kw):
        return cls(Q.n, Q.row_ptr, Q.col, Q.val, b, nranks, **kw)

    def solve(self, x0=None, tol=1e-6, maxit=1000, momentum=True, restart=True, k0=2, x_out=None,
              history=True, restart_cap=64) -> Result:
        import torch
        if x_out is None:
            x_out = torch.empty(self.n, dtype=torch.float64, device="cuda")
        rh = np.empty(maxit + 1) if history else None
        fh = np.empty(maxit + 1) if history else None
        ri = np.zeros(restart_cap, dtype=np.int64)
        p0, k_0 = _ptr(x0, np.float64)
        px, k_x = _ptr(x_out, np.float64, output=True)
        pr, k_r = _ptr(rh, np.float64, output=True)
        pf, k_f = _ptr(fh, np.float64, output=True)
        pri, k_ri = _ptr(ri, np.int64, output=True)
        arr = (ctypes.c_void_p * self.nranks)(*self.handles)
        res = ajm_result_t()
        pol = ajm_policy_t(int(bool(momentum)), int(bool(restart)), int(k0))
        _check(lib().ajm_group_solve(ctypes.cast(arr, ctypes.c_void_p), self.nranks, p0, float(tol), int(maxit), pol,
                                     px, ctypes.byref(res), pr, pf, pri, len(ri), _stream(self._stream)),
               ctypes.c_void_p(self.handles[0]))
        return _result(res, x_out, rh, fh, ri)

    def info(self, rank: int = 0) -> dict:
        return self._info(self.handles[rank])

    def load_imbalance(self, row_ptr) -> float:
        """p * max_i nnz(Q^{i,:}) / nnz(Q), the paper's load-imbalance measure."""
        rp = np.asarray(row_ptr, dtype=np.int64)
        nz = rp[self.starts[1:]] - rp[self.starts[:-1]]
        return float(self.nranks * nz.max() / max(int(rp[-1]), 1))

    def close(self):
        for h in getattr(self, "handles", []):
            if h:
                ajm_destroy(h)
        self.handles = []


def allgather_bytes(blob: bytes, group=None) -> list:
    """All ranks' connection records in rank order over torch.distributed (plumbing only)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


class ShardSolver(_ShardHandles):
    """One rank of a multi-process (one process per GPU) row-block sharded solve: create from this
    rank's rows, exchange connection records with the other ranks (``exchange(blob) -> [blobs]``,
    default torch.distributed all_gather_object), connect, then ``solve`` concurrently on every rank."""

    def __init__(self, rank: int, nranks: int, starts, row_ptr_loc, col_glob, val, b_loc, dmode="jdiag",
                 d_loc=None, int32_columns=False, segments="auto", exchange=None, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2407_03272_b200 needs a CUDA device (no CPU fallback)")
        self.rank, self.nranks = int(rank), int(nranks)
        self.starts = np.asarray(starts, dtype=np.int64)
        self.n = int(self.starts[rank + 1] - self.starts[rank])
        self._stream = stream
        flags = (AJM_INT32_COLUMNS if int32_columns else 0)
        flags |= {"auto": 0, "static": AJM_SEGMENTS_STATIC, "dynamic": AJM_SEGMENTS_DYNAMIC}[segments]
        self.handle = _shard_create(rank, nranks, self.starts, row_ptr_loc, col_glob, val, b_loc, dmode, d_loc,
                                    flags, stream)
        blobs = (exchange or allgather_bytes)(_shard_export(self.handle))
        _shard_connect(self.handle, blobs)

    def solve(self, x0=None, tol=1e-6, maxit=1000, momentum=True, restart=True, k0=2, x_out=None,
              history=True, restart_cap=64) -> Result:
        import torch
        if x_out is None:
            x_out = torch.empty(self.n, dtype=torch.float64, device="cuda")
        rh = np.empty(maxit + 1) if history else None
        fh = np.empty(maxit + 1) if history else None
        ri = np.zeros(restart_cap, dtype=np.int64)
        r = ajm_solve(self.handle, x0, tol, maxit, momentum, restart, k0, x_out, rh, fh, ri, self._stream)
        return _result(r, x_out, rh, fh, ri)

    def info(self) -> dict:
        return self._info(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            ajm_destroy(self.handle)
            self.handle = None
