"""CPU oracle for the HPL hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product path
(``paper_2304_10397_b200`` and ``libhpl.so``) never imports, links or calls
it, and it shares no code with the CUDA path (see ``hpl_oracle.c`` header).

The arithmetic lives in ``hpl_oracle.c`` (plain C, fp64, no FMA contraction);
this module only compiles it with gcc and marshals numpy arrays through ctypes.
Every function cites the passage it follows in the C source.

Parity pins (tests/test_oracle_pins.py) tie it to things other than itself:
the public SplitMix64 test vector, exact-rational brute force at n <= 8,
Cramer's rule, P·L·U == A within the LU backward-error bound, LAPACK dgetrf
pivots, closed-form residual cases and the invariants of SPEC.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hpl_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

EPS = 2.0 ** -53  # reading A4: HPL's eps is the unit roundoff 2^-53


def build(force: bool = False) -> str:
    """Compile hpl_oracle.c into liboracle.so (gcc, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            i64, u64, dp, ip = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p
            L.oracle_splitmix64.restype = u64
            L.oracle_splitmix64.argtypes = [u64, u64]
            L.oracle_gen_entry.restype = ctypes.c_double
            L.oracle_gen_entry.argtypes = [u64, i64, i64, i64]
            L.oracle_generate.restype = None
            L.oracle_generate.argtypes = [u64, i64, dp, i64, dp]
            L.oracle_getrf.restype = i64
            L.oracle_getrf.argtypes = [i64, i64, dp, i64, ip]
            L.oracle_laswp.restype = None
            L.oracle_laswp.argtypes = [dp, i64, i64, i64, i64, i64, ip]
            L.oracle_trsm_llnu.restype = None
            L.oracle_trsm_llnu.argtypes = [i64, i64, dp, i64, dp, i64]
            L.oracle_gemm_update.restype = None
            L.oracle_gemm_update.argtypes = [i64, i64, i64, dp, i64, dp, i64, dp, i64]
            L.oracle_getrs.restype = None
            L.oracle_getrs.argtypes = [i64, dp, i64, ip, dp, dp]
            L.oracle_back_solve.restype = i64
            L.oracle_back_solve.argtypes = [i64, dp, i64, dp, dp]
            L.oracle_residual.restype = ctypes.c_double
            L.oracle_residual.argtypes = [i64, dp, i64, dp, dp, dp]
            L.oracle_residual_seeded.restype = ctypes.c_double
            L.oracle_residual_seeded.argtypes = [i64, u64, dp, dp]
            L.oracle_run.restype = i64
            L.oracle_run.argtypes = [i64, u64, dp, ip, ctypes.POINTER(ctypes.c_double), dp]
            L.oracle_maxloc.restype = i64
            L.oracle_maxloc.argtypes = [i64, dp, ip]
            L.oracle_residual_rows.restype = None
            L.oracle_residual_rows.argtypes = [i64, u64, dp, i64, ip, dp, dp]
            L.oracle_set_threads.restype = None
            L.oracle_set_threads.argtypes = [ctypes.c_int]
            L.oracle_num_threads.restype = ctypes.c_int
            L.oracle_num_threads.argtypes = []
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def splitmix64(seed: int, k: int) -> int:
    return int(lib().oracle_splitmix64(seed & (2**64 - 1), k & (2**64 - 1)))


def gen_entry(seed: int, N: int, i: int, j: int) -> float:
    """A0[i][j] (j < N) or b0[i] (j == N) of the seeded system (reading A6)."""
    return float(lib().oracle_gen_entry(seed, N, i, j))


def generate(seed: int, N: int):
    """(A0, b0): the seeded N x N system, A0 row-major numpy array."""
    A = np.empty((N, N), dtype=np.float64)
    b = np.empty(N, dtype=np.float64)
    lib().oracle_generate(seed, N, _p(A), N, _p(b))
    return A, b


def getrf(A):
    """GEPP of an M x N matrix (dgetf2 semantics).  Returns (LU, ipiv, info);
    info = -1 on success, else the first column with an exact zero pivot."""
    LU = _f64c(A).copy()
    M, N = LU.shape
    ipiv = np.zeros(min(M, N), dtype=np.int64)
    info = lib().oracle_getrf(M, N, _p(LU), N, _p(ipiv))
    return LU, ipiv, int(info)


def laswp(A, k0: int, k1: int, ipiv, c0: int = 0, c1: int | None = None):
    """Apply swaps k0..k1-1 of ipiv, in order, to columns [c0, c1) of A (copy)."""
    A = _f64c(A).copy()
    ipiv = np.ascontiguousarray(ipiv, dtype=np.int64)
    c1 = A.shape[1] if c1 is None else c1
    lib().oracle_laswp(_p(A), A.shape[1], c0, c1, k0, k1, _p(ipiv))
    return A


def trsm_llnu(L, B):
    """B <- L^{-1} B with L unit lower triangular (strict upper ignored)."""
    L = _f64c(L)
    B = _f64c(B).copy()
    n, m = B.shape
    lib().oracle_trsm_llnu(n, m, _p(L), L.shape[1], _p(B), m)
    return B


def gemm_update(C, A, B):
    """C - A @ B with each dot product accumulated in ascending k order."""
    C = _f64c(C).copy()
    A = _f64c(A)
    B = _f64c(B)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2 and C.shape == (m, n)
    lib().oracle_gemm_update(m, n, k, _p(A), k, _p(B), n, _p(C), n)
    return C


def getrs(LU, ipiv, b):
    LU = _f64c(LU)
    ipiv = np.ascontiguousarray(ipiv, dtype=np.int64)
    b = _f64c(b)
    N = LU.shape[0]
    x = np.empty(N, dtype=np.float64)
    lib().oracle_getrs(N, _p(LU), LU.shape[1], _p(ipiv), _p(b), _p(x))
    return x


def back_solve(U, y):
    U = _f64c(U)
    y = _f64c(y)
    N = U.shape[0]
    x = np.empty(N, dtype=np.float64)
    info = lib().oracle_back_solve(N, _p(U), U.shape[1], _p(y), _p(x))
    return x, int(info)


def residual(A0, x, b0):
    """HPL scaled residual and (rinf, anorm, xnorm, bnorm) for an explicit system."""
    A0 = _f64c(A0)
    x = _f64c(x)
    b0 = _f64c(b0)
    out = np.zeros(4, dtype=np.float64)
    r = lib().oracle_residual(A0.shape[0], _p(A0), A0.shape[1], _p(x), _p(b0), _p(out))
    return float(r), out


def residual_seeded(N: int, seed: int, x):
    x = _f64c(x)
    out = np.zeros(4, dtype=np.float64)
    r = lib().oracle_residual_seeded(N, seed, _p(x), _p(out))
    return float(r), out


def run(N: int, seed: int, want_lu: bool = False):
    """Full oracle HPL run.  Returns dict(x, ipiv, resid, info[, LU])."""
    x = np.zeros(N, dtype=np.float64)
    ipiv = np.zeros(N, dtype=np.int64)
    resid = ctypes.c_double(float("nan"))
    LU = np.empty((N, N), dtype=np.float64) if want_lu else None
    info = lib().oracle_run(N, seed, _p(x), _p(ipiv), ctypes.byref(resid),
                            _p(LU) if want_lu else None)
    if info == -2:
        raise MemoryError("oracle_run: allocation failed")
    out = dict(x=x, ipiv=ipiv, resid=float(resid.value), info=int(info))
    if want_lu:
        out["LU"] = LU
    return out


def residual_rows(N: int, seed: int, x, rows):
    """(r, rowsum|A0|) for the given global rows of the seeded system."""
    x = _f64c(x)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    r = np.empty(len(rows), dtype=np.float64)
    a = np.empty(len(rows), dtype=np.float64)
    lib().oracle_residual_rows(N, seed, _p(x), len(rows), _p(rows), _p(r), _p(a))
    return r, a


def maxloc(absval, rows):
    """(value, row) of the pivot winner: max |v|, ties -> smallest row."""
    a = _f64c(absval)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    k = int(lib().oracle_maxloc(len(a), _p(a), _p(r)))
    return float(a[k]), int(r[k])


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())
