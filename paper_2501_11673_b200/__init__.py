"""paper_2501_11673_b200 -- B200-native Kaczmarz++ / CD++ hot path (arXiv 2501.11673).

Thin Python binding over the C ABI in ``include/kpp.h`` (``libkpp.so``, built in-tree by
``build.py`` for sm_100a).  Argument marshalling only: every step of the method runs in
the library's CUDA kernels.  PyTorch provides device memory and streams.  There is no
CPU fallback: without the library or a CUDA device every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import build as _build

__all__ = [
    "KppError", "Ctx", "SolveResult", "kpp_setup", "cdpp_setup", "kpp_solve", "cdpp_solve",
    "kpp_destroy", "kpp_get_unique_id", "kpp_setup_dist", "cdpp_setup_dist", "load_library",
    "OPT_ACCEL", "OPT_MEMO", "OPT_ETA", "OPT_RHO_FIXED", "OPT_FACTOR", "OPT_WINDOW",
    "OPT_PHASE1_MB", "OPT_RESIDENT", "OPT_ENGINE", "OPT_CLUSTER", "OPT_YGL", "OPT_REASSOC", "OPT_PROJ", "OPT_TMAX", "OPT_TAU", "OPT_XCHG", "OPT_RHO0", "OPT_RHO_MAX", "OPT_VRANKS",
]

OK, EINVAL, ENOMEM, ECUDA, ENCCL, ENOTPD, EDIVERGED, EMAXITER = range(8)
OPT_ACCEL, OPT_MEMO, OPT_ETA, OPT_RHO_FIXED, OPT_FACTOR, OPT_WINDOW, OPT_PHASE1_MB, OPT_RESIDENT = range(1, 9)
OPT_ENGINE = 9  # -1 auto (default); 0 persistent kernel; 1 graph of step kernels; 2 fused-exchange kernel
OPT_CLUSTER = 10  # 0: automatic; 1/2/4/8/16: forced thread-block cluster size
OPT_XCHG = 16  # column-sharded exchange: 1 fused NVLink peer exchange (default), 0 NCCL
OPT_PROJ, OPT_TMAX, OPT_TAU = 13, 14, 15  # K++ projection: 1 = sketch + LSQR (Alg 6), t_max, tau
OPT_REASSOC = 12  # CD++: 1 re-associated streaming kernel when blocks stream (default), 0 off, 2 always
OPT_VRANKS = 19  # engine 2 on one GPU: emulate P column-sharded ranks in one launch (protocol test)
OPT_RHO0, OPT_RHO_MAX = 17, 18  # initial rho (default 0); adaptive-rho upper clamp (default 0.99, Q9)
OPT_YGL = 11  # -1: automatic; 0: y = M r per cluster; 1: once per GPU (L2 gather); 4: per cluster from partials

LIB_PATH = _build.LIB
_lib = None


class KppError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class _Stats(ctypes.Structure):
    _fields_ = [("phase1_ms", ctypes.c_double), ("phase2_ms", ctypes.c_double),
                ("iter_kernel_ms", ctypes.c_double), ("n_blocks", ctypes.c_int64),
                ("n_fresh_last", ctypes.c_int64), ("iter_launches", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("grid_ctas", ctypes.c_int32),
                ("resident", ctypes.c_int32), ("cluster", ctypes.c_int32), ("m_in_smem", ctypes.c_int32),
                ("tma", ctypes.c_int32), ("ygl", ctypes.c_int32), ("reassoc", ctypes.c_int32),
                ("n_refined", ctypes.c_int64), ("rht_ms", ctypes.c_double), ("xchg", ctypes.c_int32),
                ("engine", ctypes.c_int32)]


def load_library():
    """Load libkpp.so (must have been built: ``python -m paper_2501_11673_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise KppError(ECUDA, f"{LIB_PATH} is missing: build it with paper_2501_11673_b200/build.py")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "kpp_setup": ([PP, P, i64, i64, i64, i32, f64, u64], i32),
        "cdpp_setup": ([PP, P, i64, i64, i32, f64, u64], i32),
        "kpp_solve": ([P, P, P, i64, f64, P, P, i64, P, P], i32),
        "cdpp_solve": ([P, P, P, i64, f64, P, P, i64, P, P], i32),
        "kpp_destroy": ([P], None),
        "kpp_status_str": ([i32], ctypes.c_char_p),
        "kpp_last_error": ([P], ctypes.c_char_p),
        "kpp_set_stream": ([P, P], i32),
        "kpp_set_option": ([P, i32, f64], i32),
        "kpp_get_schedule": ([P, i64, i64, P, P], i32),
        "kpp_get_block": ([P, i64, P], i32),
        "kpp_get_factor": ([P, i64, P], i32),
        "kpp_prepare": ([P, i64], i32),
        "kpp_clear_cache": ([P], i32),
        "kpp_get_rho_history": ([P, P, i64, P], i32),
        "kpp_get_stats": ([P, P], i32),
        "kpp_reset_stats": ([P], i32),
        "kpp_get_unique_id": ([P], i32),
        "kpp_setup_dist": ([PP, P, i64, i64, i64, i64, i64, i32, f64, u64, P, i32, i32], i32),
        "cdpp_setup_dist": ([PP, P, i64, i64, i64, i64, i32, f64, u64, P, i32, i32], i32),
        "kpp_version": ([], ctypes.c_char_p),
        "kpp_enable_rht": ([P], i32),
        "kpp_get_rht_matrix": ([P, P], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(status: int, handle=None, allow=(OK,)):
    if status in allow:
        return status
    L = load_library()
    msg = L.kpp_status_str(status).decode()
    if handle:
        detail = L.kpp_last_error(handle).decode()
        if detail:
            msg += f": {detail}"
    raise KppError(status, msg)


def _dev_f64(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a float64 torch.Tensor")
    return t.contiguous()


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


@dataclass
class SolveResult:
    x: torch.Tensor
    status: int
    iters: int
    res_hist: torch.Tensor  # per-checkpoint sqrt(E1/||b||^2), host fp64

    @property
    def converged(self) -> bool:
        return self.status == OK


class Ctx:
    """A kpp_ctx handle.  Keeps a reference to A (borrowed by the library)."""

    def __init__(self, handle, A: torch.Tensor, kind: str, m: int, n_local: int, s: int):
        self._h = handle
        self._A = A
        self.kind = kind
        self.m = m
        self.n = n_local
        self.s = s

    @property
    def handle(self):
        if not self._h:
            raise KppError(EINVAL, "context destroyed")
        return self._h

    def set_option(self, key: int, value: float):
        _check(load_library().kpp_set_option(self.handle, key, float(value)), self.handle)

    def set_stream(self, stream: torch.cuda.Stream | None = None):
        s = stream if stream is not None else torch.cuda.current_stream()
        _check(load_library().kpp_set_stream(self.handle, ctypes.c_void_p(s.cuda_stream)), self.handle)

    def solve(self, b, x0=None, max_iters=1000, tol=0.0, x_out=None, hist_cap=1 << 16,
              allow_maxiter=True) -> SolveResult:
        return kpp_solve(self, b, x0, max_iters, tol, x_out, hist_cap, allow_maxiter)

    def schedule(self, t0: int, count: int):
        bid = torch.zeros(count, dtype=torch.int32)
        fresh = torch.zeros(count, dtype=torch.uint8)
        _check(load_library().kpp_get_schedule(self.handle, t0, count, _ptr(bid), _ptr(fresh)), self.handle)
        return bid, fresh

    def prepare(self, iters: int):
        _check(load_library().kpp_prepare(self.handle, iters), self.handle)

    def clear_cache(self):
        """Forget every memoized block: the next solve is cold (Phase 1 for every fresh block)."""
        _check(load_library().kpp_clear_cache(self.handle), self.handle)

    def block(self, k: int) -> torch.Tensor:
        S = torch.zeros(self.s, dtype=torch.int32)
        _check(load_library().kpp_get_block(self.handle, k, _ptr(S)), self.handle)
        return S

    def factor(self, k: int) -> torch.Tensor:
        M = torch.zeros(self.s, self.s, dtype=torch.float64)
        _check(load_library().kpp_get_factor(self.handle, k, _ptr(M)), self.handle)
        return M

    def rho_history(self) -> torch.Tensor:
        L = load_library()
        n = ctypes.c_int64()
        _check(L.kpp_get_rho_history(self.handle, None, 0, ctypes.byref(n)), self.handle)
        out = torch.zeros(n.value, dtype=torch.float64)
        _check(L.kpp_get_rho_history(self.handle, _ptr(out), n.value, ctypes.byref(n)), self.handle)
        return out

    def stats(self) -> dict:
        st = _Stats()
        _check(load_library().kpp_get_stats(self.handle, ctypes.byref(st)), self.handle)
        return {k: getattr(st, k) for k, _ in _Stats._fields_}

    def reset_stats(self):
        _check(load_library().kpp_reset_stats(self.handle), self.handle)

    def enable_rht(self):
        """Randomized Hadamard preprocessing (kpp_enable_rht): later solves run on Q A (K++) or
        Q A Q^T (CD++) with the caller's b / x sizes unchanged."""
        _check(load_library().kpp_enable_rht(self.handle), self.handle)
        self._rht_dims = self._rht_shape()

    def _rht_shape(self):
        p2 = lambda v: 1 << max(0, (v - 1).bit_length())
        return (p2(self.m), self.n) if self.kind == "kpp" else (p2(self.n), p2(self.n))

    def rht_matrix(self) -> torch.Tensor:
        out = torch.zeros(*self._rht_shape(), dtype=torch.float64)
        _check(load_library().kpp_get_rht_matrix(self.handle, _ptr(out)), self.handle)
        return out

    def destroy(self):
        if self._h:
            load_library().kpp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def _require_cuda(A: torch.Tensor):
    if not torch.cuda.is_available() or not A.is_cuda:
        raise KppError(EINVAL, "A must be a CUDA tensor (no CPU fallback)")


def kpp_setup(A: torch.Tensor, block_size: int, lam: float = 1e-8, seed: int = 0) -> Ctx:
    """Kaczmarz++ context for a general m x n fp64 CUDA matrix (row-major)."""
    A = _dev_f64(A, "A")
    _require_cuda(A)
    L = load_library()
    h = ctypes.c_void_p()
    m, n = A.shape
    _check(L.kpp_setup(ctypes.byref(h), _ptr(A), m, n, A.stride(0), block_size, lam, seed))
    return Ctx(h, A, "kpp", m, n, block_size)


def cdpp_setup(A: torch.Tensor, block_size: int, lam: float = 1e-8, seed: int = 0) -> Ctx:
    """CD++ context for a symmetric PSD n x n fp64 CUDA matrix."""
    A = _dev_f64(A, "A")
    _require_cuda(A)
    L = load_library()
    h = ctypes.c_void_p()
    n = A.shape[0]
    if A.shape[1] != n:
        raise KppError(EINVAL, "CD++ needs a square matrix")
    _check(L.cdpp_setup(ctypes.byref(h), _ptr(A), n, A.stride(0), block_size, lam, seed))
    return Ctx(h, A, "cdpp", n, n, block_size)


def kpp_solve(ctx: Ctx, b: torch.Tensor, x0: torch.Tensor | None = None, max_iters: int = 1000,
              tol: float = 0.0, x_out: torch.Tensor | None = None, hist_cap: int = 1 << 16,
              allow_maxiter: bool = True) -> SolveResult:
    """One solve.  b / x0 / x_out may live on the device or (pinned or pageable) host."""
    b = _dev_f64(b, "b")
    if x0 is not None:
        x0 = _dev_f64(x0, "x0")
    if x_out is None:
        x_out = torch.empty(ctx.n, dtype=torch.float64, device=b.device)
    # the C ABI takes bare pointers: sizes are checked here (b has the m rows of the problem --
    # the caller's m with RHT, the full m on a column-sharded context; x0 / x_out the n local columns)
    if b.numel() != ctx.m:
        raise KppError(EINVAL, f"b has {b.numel()} entries, expected m = {ctx.m}")
    if x0 is not None and x0.numel() != ctx.n:
        raise KppError(EINVAL, f"x0 has {x0.numel()} entries, expected n = {ctx.n}")
    if not isinstance(x_out, torch.Tensor) or x_out.dtype != torch.float64 or not x_out.is_contiguous() \
            or x_out.numel() != ctx.n:
        raise KppError(EINVAL, f"x_out must be a contiguous float64 tensor of n = {ctx.n} entries")
    L = load_library()
    hist = torch.zeros(max(hist_cap, 1), dtype=torch.float64)
    nh, it = ctypes.c_int64(), ctypes.c_int64()
    st = L.kpp_solve(ctx.handle, _ptr(b), _ptr(x0) if x0 is not None else None, int(max_iters),
                     float(tol), _ptr(x_out), _ptr(hist), hist_cap, ctypes.byref(nh), ctypes.byref(it))
    _check(st, ctx.handle, allow=(OK, EMAXITER) if allow_maxiter else (OK,))
    k = min(nh.value, hist_cap)
    return SolveResult(x_out, st, it.value, hist[:k].clone())


def cdpp_solve(ctx: Ctx, b, x0=None, max_iters=1000, tol=0.0, x_out=None, hist_cap=1 << 16,
               allow_maxiter=True) -> SolveResult:
    if ctx.kind != "cdpp":
        raise KppError(EINVAL, "cdpp_solve needs a CD++ context")
    return kpp_solve(ctx, b, x0, max_iters, tol, x_out, hist_cap, allow_maxiter)


def kpp_destroy(ctx: Ctx):
    ctx.destroy()


def kpp_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(load_library().kpp_get_unique_id(buf))
    return bytes(buf)


def _dist_setup(fn, A_slab, m, n_global, col_begin, col_end, block_size, lam, seed, uid, rank, nranks,
                kind):
    A_slab = _dev_f64(A_slab, "A_slab")
    _require_cuda(A_slab)
    L = load_library()
    h = ctypes.c_void_p()
    idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    if kind == "kpp":
        st = L.kpp_setup_dist(ctypes.byref(h), _ptr(A_slab), m, n_global, col_begin, col_end,
                              A_slab.stride(0), block_size, lam, seed, idbuf, rank, nranks)
    else:
        st = L.cdpp_setup_dist(ctypes.byref(h), _ptr(A_slab), n_global, col_begin, col_end,
                               A_slab.stride(0), block_size, lam, seed, idbuf, rank, nranks)
    _check(st)
    return Ctx(h, A_slab, kind, m, col_end - col_begin, block_size)


def kpp_setup_dist(A_slab, m, n_global, col_begin, col_end, block_size, lam, seed, uid, rank, nranks):
    """Column-sharded Kaczmarz++: this rank owns A[:, col_begin:col_end]."""
    return _dist_setup(None, A_slab, m, n_global, col_begin, col_end, block_size, lam, seed, uid, rank,
                       nranks, "kpp")


def cdpp_setup_dist(A_slab, n, col_begin, col_end, block_size, lam, seed, uid, rank, nranks):
    """Column-sharded CD++: this rank owns A[:, col_begin:col_end] of the symmetric A."""
    return _dist_setup(None, A_slab, n, n, col_begin, col_end, block_size, lam, seed, uid, rank,
                       nranks, "cdpp")


def column_slabs(n: int, nranks: int):
    """Contiguous column slabs [p*n/P, (p+1)*n/P); host-side partition logic."""
    return [(p * n // nranks, (p + 1) * n // nranks) for p in range(nranks)]
