"""CPU oracle for the Kaczmarz++ / CD++ hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(``paper_2501_11673_b200``) never imports it and shares no code with it.

This module is a thin ctypes loader over ``kpp_oracle.cpp`` (plain C++17, fp64,
sequential sums, -ffp-contract=off).  See ``kpp_oracle.h`` for the per-function
citations of PAPER.md and the pin status of each function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kpp_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, ENOTPD, EDIVERGED, EMAXITER = 0, 1, 5, 6, 7
HOUSEHOLDER, GRAM = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so in-tree (g++, -O2 -ffp-contract=off, OpenMP over outputs)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "kpp_oracle.h"))
    ):
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB, _SRC]
        subprocess.check_call(cmd)
    return _LIB


class _Opts(ctypes.Structure):
    _fields_ = [("accel", ctypes.c_int32), ("memo", ctypes.c_int32),
                ("eta_override", ctypes.c_double), ("rho_fixed", ctypes.c_double),
                ("factor", ctypes.c_int32), ("reverse", ctypes.c_int32),
                ("threads", ctypes.c_int32), ("proj", ctypes.c_int32), ("tmax", ctypes.c_int32),
                ("tau", ctypes.c_int32), ("rho0", ctypes.c_double), ("rho_max", ctypes.c_double),
                ("timing", ctypes.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, u64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        L.ora_philox4x32_10.argtypes = [P, P, P]
        L.ora_fresh_block.argtypes = [u64, i64, i32, i64, P]
        L.ora_schedule.argtypes = [u64, f64, i32, i64, P, P]
        L.ora_schedule.restype = i64
        L.ora_kpp_C.argtypes = [i64, i64, i32]
        L.ora_kpp_C.restype = f64
        L.ora_cdpp_C.argtypes = [i64, i32]
        L.ora_cdpp_C.restype = f64
        L.ora_kpp_factor.argtypes = [P, i64, i64, P, i32, f64, i32, i32, P]
        L.ora_cdpp_factor.argtypes = [P, i64, P, i32, f64, i32, P]
        run_args = [P, i64, i64, i64, P, P, i32, f64, u64, i64, f64, ctypes.POINTER(_Opts),
                    P, P, P, i64, P, P, P]
        L.ora_kpp_run.argtypes = run_args
        L.ora_cdpp_run.argtypes = [P, i64, i64, P, P, i32, f64, u64, i64, f64,
                                   ctypes.POINTER(_Opts), P, P, P, i64, P, P, P]
        L.ora_rho_update.argtypes = [i64, f64, f64, f64, i64, P, P]
        L.ora_srht.argtypes = [u64, i64, i32, P, P]
        L.ora_sketch_factor.argtypes = [P, i64, i64, P, i32, f64, u64, i32, P]
        L.ora_lsqr_proj.argtypes = [P, i64, i64, P, i32, f64, P, P, i32, P]
        L.ora_next_pow2.argtypes = [i64]
        L.ora_next_pow2.restype = i64
        L.ora_rht_signs.argtypes = [u64, i64, P]
        L.ora_fht.argtypes = [P, i64]
        L.ora_rht_rows.argtypes = [P, i64, i64, i64, P, u64, P, P]
        L.ora_rht_sym.argtypes = [P, i64, i64, P, u64, P, P]
        L.ora_rht_vec.argtypes = [P, i64, i64, u64, i32, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().ora_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def fresh_block(seed: int, pop: int, s: int, k: int) -> np.ndarray:
    S = np.zeros(s, dtype=np.int32)
    lib().ora_fresh_block(seed, pop, s, k, _p(S))
    return S


def kpp_C(m, n, s):
    return lib().ora_kpp_C(m, n, s)


def cdpp_C(n, s):
    return lib().ora_cdpp_C(n, s)


def schedule(seed: int, C: float, T: int, memo: bool = True):
    bid = np.zeros(T, dtype=np.int32)
    fresh = np.zeros(T, dtype=np.uint8)
    nb = lib().ora_schedule(seed, C, int(memo), T, _p(bid), _p(fresh))
    return bid, fresh, int(nb)


def kpp_factor(A, S, lam, mode=HOUSEHOLDER, reverse=False):
    A = _f64(A)
    S = np.ascontiguousarray(S, dtype=np.int32)
    s = S.size
    R = np.zeros((s, s))
    rc = lib().ora_kpp_factor(_p(A), A.shape[1], A.shape[1], _p(S), s, lam, mode, int(reverse), _p(R))
    if rc != OK:
        raise RuntimeError(f"oracle factor failed: {rc}")
    return R


def cdpp_factor(A, S, lam, reverse=False):
    A = _f64(A)
    S = np.ascontiguousarray(S, dtype=np.int32)
    s = S.size
    R = np.zeros((s, s))
    rc = lib().ora_cdpp_factor(_p(A), A.shape[1], _p(S), s, lam, int(reverse), _p(R))
    if rc != OK:
        raise RuntimeError(f"oracle factor failed: {rc}")
    return R


def rho_update(i, rhat_prev, E0, E1, zeta):
    rh = ctypes.c_double()
    rho = ctypes.c_double()
    lib().ora_rho_update(i, rhat_prev, E0, E1, zeta, ctypes.byref(rh), ctypes.byref(rho))
    return rh.value, rho.value


@dataclass
class Result:
    x: np.ndarray
    status: int
    iters: int
    nfresh: int
    hist_res: np.ndarray
    hist_rho: np.ndarray


def _run(cd, A, b, s, lam, seed, max_iters, tol, x0, accel, memo, eta, rho_fixed, factor,
         reverse, threads, hist_cap, proj=0, tmax=8, tau=0, rho0=0.0, rho_max=0.99, timing=None):
    A = _f64(A)
    b = _f64(b)
    n = A.shape[1]
    m = A.shape[0]
    x = np.zeros(n)
    x0p = None if x0 is None else _p(_f64(x0))
    x0keep = None if x0 is None else _f64(x0)
    if x0keep is not None:
        x0p = _p(x0keep)
    hr = np.zeros(hist_cap)
    hp = np.zeros(hist_cap)
    nh, it, nf = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    o = _Opts(int(accel), int(memo), -1.0 if eta is None else float(eta),
              -1.0 if rho_fixed is None else float(rho_fixed), int(factor), int(reverse),
              int(threads), int(proj), int(tmax), int(tau), float(rho0), float(rho_max),
              ctypes.c_void_p(timing.ctypes.data) if timing is not None else None)
    if cd:
        rc = lib().ora_cdpp_run(_p(A), n, n, _p(b), x0p, s, lam, seed, max_iters, tol,
                                ctypes.byref(o), _p(x), _p(hr), _p(hp), hist_cap,
                                ctypes.byref(nh), ctypes.byref(it), ctypes.byref(nf))
    else:
        rc = lib().ora_kpp_run(_p(A), m, n, n, _p(b), x0p, s, lam, seed, max_iters, tol,
                               ctypes.byref(o), _p(x), _p(hr), _p(hp), hist_cap,
                               ctypes.byref(nh), ctypes.byref(it), ctypes.byref(nf))
    k = min(nh.value, hist_cap)
    return Result(x, rc, it.value, nf.value, hr[:k].copy(), hp[:k].copy())


def kpp_run(A, b, s, lam=1e-8, seed=0, max_iters=100, tol=0.0, x0=None, accel=True, memo=True,
            eta=None, rho_fixed=None, factor=HOUSEHOLDER, reverse=False, threads=1,
            hist_cap=1 << 16, proj=0, tmax=8, tau=0, rho0=0.0, rho_max=0.99, timing=None) -> Result:
    """Kaczmarz++ (Alg 5; proj=0 exact projections (K++(Cholesky)), proj=1 sketch + LSQR, Alg 6)
    -- see kpp_oracle.h."""
    return _run(False, A, b, s, lam, seed, max_iters, tol, x0, accel, memo, eta, rho_fixed,
                factor, reverse, threads, hist_cap, proj, tmax, tau, rho0, rho_max, timing)


def cdpp_run(A, b, s, lam=1e-8, seed=0, max_iters=100, tol=0.0, x0=None, accel=True, memo=True,
             eta=None, rho_fixed=None, reverse=False, threads=1, hist_cap=1 << 16, rho0=0.0,
             rho_max=0.99, timing=None) -> Result:
    """CD++ (Alg 3 without SymFHT) -- see kpp_oracle.h."""
    return _run(True, A, b, s, lam, seed, max_iters, tol, x0, accel, memo, eta, rho_fixed,
                HOUSEHOLDER, reverse, threads, hist_cap, rho0=rho0, rho_max=rho_max, timing=timing)


# ---------------------------------------------------------------- RHT
def next_pow2(n: int) -> int:
    return int(lib().ora_next_pow2(n))


def rht_signs(seed: int, n: int) -> np.ndarray:
    d = np.zeros(n, dtype=np.int8)
    lib().ora_rht_signs(seed, n, _p(d))
    return d


def fht(v) -> np.ndarray:
    w = _f64(v).copy()
    lib().ora_fht(_p(w), w.shape[0])
    return w


def rht_rows(A, b, seed: int):
    """K++ preprocessing: (H D [A; 0], H D [b; 0]) with m2 = next power of 2 rows."""
    A = _f64(A)
    m, n = A.shape
    m2 = next_pow2(m)
    At = np.zeros((m2, n))
    bt = np.zeros(m2)
    lib().ora_rht_rows(_p(A), m, n, n, _p(_f64(b)), seed, _p(At), _p(bt))
    return At, bt


def rht_sym(A, b, seed: int):
    """CD++ preprocessing: (H D A_pad D H, H D [b; 0])."""
    A = _f64(A)
    n = A.shape[0]
    n2 = next_pow2(n)
    At = np.zeros((n2, n2))
    bt = np.zeros(n2)
    lib().ora_rht_sym(_p(A), n, n, _p(_f64(b)), seed, _p(At), _p(bt))
    return At, bt


def rht_vec(v, n: int, n2: int, seed: int, forward: bool) -> np.ndarray:
    """forward: H D [v; 0] (n2 values); backward: (D H v)[:n] (Alg 3 l.16)."""
    v = _f64(v)
    out = np.zeros(n2 if forward else n)
    lib().ora_rht_vec(_p(v), n, n2, seed, int(forward), _p(out))
    return out


def kpp_run_rht(A, b, s, seed=0, **kw) -> Result:
    """Alg 5 with its preprocessing lines 2-3: solve H D A x = H D b (same x)."""
    At, bt = rht_rows(A, b, seed)
    return kpp_run(At, bt, s, seed=seed, **kw)


def cdpp_run_rht(A, b, s, seed=0, x0=None, **kw) -> Result:
    """Alg 3 with lines 2-3 and the back-rotation of line 16: x = D H xt."""
    n = A.shape[0]
    n2 = next_pow2(n)
    At, bt = rht_sym(A, b, seed)
    xt0 = None if x0 is None else rht_vec(x0, n, n2, seed, True)
    r = cdpp_run(At, bt, s, seed=seed, x0=xt0, **kw)
    r.x = rht_vec(r.x, n, n2, seed, False)
    return r


# ---------------------------------------------------------------- sketch + LSQR (NEXT-2)
def srht(seed: int, n: int, tau: int):
    n2 = next_pow2(n)
    d = np.zeros(n2)
    T = np.zeros(tau, dtype=np.int32)
    lib().ora_srht(seed, n, tau, _p(d), _p(T))
    return d, T


def sketch_factor(A, S, lam, seed, tau):
    A = _f64(A)
    S = np.ascontiguousarray(S, dtype=np.int32)
    s = S.shape[0]
    R = np.zeros((s, s))
    rc = lib().ora_sketch_factor(_p(A), A.shape[1], A.shape[1], _p(S), s, lam, seed, tau, _p(R))
    if rc != OK:
        raise RuntimeError(f"sketch factor failed: {rc}")
    return R


def lsqr_proj(A, S, lam, R, r, tmax):
    A = _f64(A)
    S = np.ascontiguousarray(S, dtype=np.int32)
    w = np.zeros(A.shape[1])
    lib().ora_lsqr_proj(_p(A), A.shape[1], A.shape[1], _p(S), S.shape[0], lam, _p(_f64(R)), _p(_f64(r)),
                        tmax, _p(w))
    return w
