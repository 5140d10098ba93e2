"""Thin Python layer over libhpl.so with the C ABI's names (marshalling only).

    ctx = hpl_init(N, NB, P, Q, seed)        # device-generated system
    hpl_factor(ctx); x = hpl_solve(ctx); r = hpl_residual(ctx); hpl_free(ctx)

Kernel-level entry points (hplk_*) take and return numpy arrays; they run
the exact kernels of the hot path on copies of the inputs (parity tests).
"""
from __future__ import annotations

import ctypes

import numpy as np

from ._lib import lib, ptr

STATUS = {0: "HPL_OK", 1: "HPL_ERR_ARG", 2: "HPL_ERR_STATE", 3: "HPL_ERR_OOM",
          4: "HPL_ERR_CUDA", 5: "HPL_ERR_NCCL", 6: "HPL_ERR_SINGULAR", 7: "HPL_ERR_PEER"}


class HplError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class HplSingular(HplError):
    def __init__(self, status, msg, column):
        super().__init__(status, msg)
        self.column = column


class Ctx:
    """Owns an hpl_ctx*.  Use as a context manager or call hpl_free."""

    def __init__(self, handle: int, N: int, NB: int, P: int, Q: int, seed: int):
        self.h = ctypes.c_void_p(handle)
        self.N, self.NB, self.P, self.Q, self.seed = N, NB, P, Q, seed

    def check(self, st: int):
        if st == 0:
            return
        msg = lib.hpl_last_error(self.h).decode(errors="replace")
        if st == 6:
            raise HplSingular(st, msg, int(lib.hpl_singular_column(self.h)))
        raise HplError(st, msg)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        hpl_free(self)

    @property
    def local_shape(self):
        r, c = ctypes.c_int64(), ctypes.c_int64()
        self.check(lib.hpl_local_shape(self.h, ctypes.byref(r), ctypes.byref(c)))
        return int(r.value), int(c.value)


def hpl_init(N: int, NB: int, P: int = 1, Q: int = 1, seed: int = 42) -> Ctx:
    h = ctypes.c_void_p()
    st = lib.hpl_init(N, NB, P, Q, seed, ctypes.byref(h))
    if st != 0:
        msg = lib.hpl_last_error(h).decode(errors="replace") if h.value else "invalid argument"
        if h.value:
            lib.hpl_free(h)
        raise HplError(st, msg)
    return Ctx(h.value, N, NB, P, Q, seed)


def hpl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib.hpl_get_unique_id(buf)
    if st != 0:
        raise HplError(st, "hpl_get_unique_id failed")
    return buf.raw


def hpl_init_dist(N: int, NB: int, P: int, Q: int, seed: int, rank: int, nranks: int,
                  unique_id: bytes, device: int) -> Ctx:
    h = ctypes.c_void_p()
    idbuf = ctypes.create_string_buffer(unique_id, 128)
    st = lib.hpl_init_dist(N, NB, P, Q, seed, rank, nranks, idbuf, device, ctypes.byref(h))
    if st != 0:
        msg = lib.hpl_last_error(h).decode(errors="replace") if h.value else "invalid argument"
        if h.value:
            lib.hpl_free(h)
        raise HplError(st, msg)
    return Ctx(h.value, N, NB, P, Q, seed)


def hpl_init_loopback(N: int, NB: int, P: int, Q: int, seed: int = 42, device: int = 0) -> list:
    """The P*Q rank contexts of one grid on one device of this process
    (include/hpl.h hpl_init_loopback); drive them with run_ranks."""
    nr = P * Q
    hs = (ctypes.c_void_p * nr)()
    st = lib.hpl_init_loopback(N, NB, P, Q, seed, device, hs)
    ctxs = [Ctx(h, N, NB, P, Q, seed) if h else None for h in hs]
    if st != 0:
        msg = next((lib.hpl_last_error(c.h).decode(errors="replace") for c in ctxs
                    if c is not None and lib.hpl_last_error(c.h)), "")
        if not msg and st == 2:
            msg = ("needs CUDA_MODULE_LOADING=EAGER and CUDA_DEVICE_MAX_CONNECTIONS >= 3*P*Q "
                   "before CUDA initialises")
        for c in ctxs:
            if c is not None:
                hpl_free(c)
        raise HplError(st, msg or "invalid argument")
    return ctxs


def run_ranks(fn, ctxs: list) -> list:
    """Call fn(ctx) for every rank context concurrently, one host thread per
    rank (ctypes releases the GIL during the library call), and return the
    results in rank order; the first exception raised by a rank is re-raised
    after every thread has finished."""
    import threading
    out = [None] * len(ctxs)
    err = [None] * len(ctxs)

    def body(r):
        try:
            out[r] = fn(ctxs[r])
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    bad = [(r, e) for r, e in enumerate(err) if e is not None]
    if bad:
        # the first failing rank's exception, with every rank's message attached
        e = bad[0][1]
        if len(bad) > 1 and isinstance(e, HplError):
            e.args = (e.args[0] + " | " + "; ".join(f"rank {r}: {x}" for r, x in bad[1:]),)
        raise e
    return out


def hpl_factor(ctx: Ctx) -> None:
    ctx.check(lib.hpl_factor(ctx.h))


def hpl_solve(ctx: Ctx, want_x: bool = True):
    if not want_x:
        ctx.check(lib.hpl_solve(ctx.h, None))
        return None
    x = np.empty(ctx.N, dtype=np.float64)
    ctx.check(lib.hpl_solve(ctx.h, ptr(x)))
    return x


def hpl_residual(ctx: Ctx) -> float:
    r = ctypes.c_double()
    ctx.check(lib.hpl_residual(ctx.h, ctypes.byref(r)))
    return float(r.value)


def hpl_regenerate(ctx: Ctx) -> None:
    ctx.check(lib.hpl_regenerate(ctx.h))


def hpl_load_local(ctx: Ctx, host: np.ndarray) -> None:
    host = np.ascontiguousarray(host, dtype=np.float64)
    rows, cols = ctx.local_shape
    if host.shape != (rows, cols):
        raise ValueError(f"expected local block {(rows, cols)}, got {host.shape}")
    ctx.check(lib.hpl_load_local(ctx.h, ptr(host), cols))


def hpl_load_factor(ctx: Ctx, host: np.ndarray) -> None:
    """hpl_load_local + hpl_factor with the copy overlapped (include/hpl.h);
    pin `host` with hpl_pin_host for the overlap."""
    if host.dtype != np.float64 or not host.flags.c_contiguous:
        raise ValueError("host must be a C-contiguous float64 array")
    rows, cols = ctx.local_shape
    if host.shape != (rows, cols):
        raise ValueError(f"expected local block {(rows, cols)}, got {host.shape}")
    ctx.check(lib.hpl_load_factor(ctx.h, ptr(host), cols))


def hpl_free(ctx: Ctx) -> None:
    if ctx.h is not None and ctx.h.value:
        lib.hpl_free(ctx.h)
        ctx.h = ctypes.c_void_p()


def hpl_get_ipiv(ctx: Ctx) -> np.ndarray:
    ip = np.empty(ctx.N, dtype=np.int64)
    ctx.check(lib.hpl_get_ipiv(ctx.h, ptr(ip)))
    return ip


def hpl_get_local(ctx: Ctx) -> np.ndarray:
    rows, cols = ctx.local_shape
    out = np.empty((rows, cols), dtype=np.float64)
    ctx.check(lib.hpl_get_local(ctx.h, ptr(out), cols))
    return out


def hpl_get_timeline(ctx: Ctx, cap: int = 1 << 16) -> np.ndarray:
    buf = np.zeros((cap, 6), dtype=np.float64)
    n = lib.hpl_get_timeline(ctx.h, ptr(buf), cap)
    return buf[:n]


def hpl_get_fact_detail(ctx: Ctx, cap: int = 1 << 16) -> np.ndarray:
    """[wait, fact_local, lbcast_plan] ms per iteration (see include/hpl.h)."""
    buf = np.zeros((cap, 3), dtype=np.float64)
    n = lib.hpl_get_fact_detail(ctx.h, ptr(buf), cap)
    return buf[:n]


def hpl_set_timing(ctx: Ctx, enable: bool = True) -> None:
    ctx.check(lib.hpl_set_timing(ctx.h, 1 if enable else 0))


def hpl_set_option(ctx: Ctx, name: str, value: int) -> None:
    ctx.check(lib.hpl_set_option(ctx.h, name.encode(), int(value)))


def hpl_launch_count(ctx: Ctx) -> int:
    return int(lib.hpl_launch_count(ctx.h))


def hpl_last_timing(ctx: Ctx) -> dict:
    """Device-timed results of the last factor/solve (CUDA events)."""
    o = np.zeros(6, dtype=np.float64)
    ctx.check(lib.hpl_last_timing(ctx.h, ptr(o)))
    return dict(factor_ms=o[0], solve_ms=o[1], dgemm_launches=int(o[2]), dgemm_ms=o[3],
                dgemm_flop=o[4], launches=int(o[5]))


def hpl_phase_stats(ctx: Ctx) -> dict:
    """Per-phase totals of the last factor/solve (include/hpl.h hpl_phase_stats)."""
    o = np.zeros(12, dtype=np.float64)
    ctx.check(lib.hpl_phase_stats(ctx.h, ptr(o)))
    return dict(laswp_ms=o[0], laswp_bytes=o[1], trsm_ms=o[2], trsm_flop=o[3], fact_ms=o[4],
                solve_ms=o[5], solve_bytes=o[6], dgemm_ms=o[7], h2d_ms=o[8], h2d_bytes=o[9],
                pipelined_ms=o[10], pipelined_iters=int(o[11]))


def hpl_plan_iteration(N: int, NB: int, P: int, Q: int, myrow: int, mycol: int, j: int) -> dict:
    """Host-only bookkeeping of iteration j on process (myrow, mycol)."""
    o = np.zeros(8, dtype=np.int64)
    st = lib.hpl_plan_iteration(N, NB, P, Q, myrow, mycol, j, ptr(o))
    if st != 0:
        raise HplError(st, "hpl_plan_iteration: invalid arguments")
    return dict(lr0=int(o[0]), lct=int(o[1]), la=(int(o[2]), int(o[3])), rest=(int(o[4]), int(o[5])),
                lpanel=int(o[6]), jb=int(o[7]))


def hpl_plan_fact(N: int, NB: int, P: int, Q: int, myrow: int, j: int,
                  gather_rows: int = 65536, gather_ms: float = 8.0) -> dict:
    """Host-only bookkeeping of panel j's FACT on process row myrow (P > 1:
    distributed leaf or gathered FACT, decided from global sizes)."""
    o = np.zeros(5, dtype=np.int64)
    st = lib.hpl_plan_fact(N, NB, P, Q, myrow, j, gather_rows, float(gather_ms), ptr(o))
    if st != 0:
        raise HplError(st, "hpl_plan_fact: invalid arguments")
    return dict(mode=int(o[0]), rows=int(o[1]), lrL0=int(o[2]), mL=int(o[3]), ldp=int(o[4]))


def hpl_pin_host(arr: np.ndarray, pin: bool = True) -> bool:
    """Page-lock a host array for DMA-speed copies; returns False if refused."""
    return lib.hpl_pin_host(ptr(arr), arr.nbytes, 1 if pin else 0) == 0


# ---------------------------------------------------------------- kernel-level
def _k(st: int, what: str):
    if st != 0:
        raise HplError(4 if st > 0 else 1, f"{what} returned {st}")


def hplk_dgemm_update(C, A, B, cfg: int = -1):
    """C - A @ B on the DMMA kernel (A passed as given; stored col-major)."""
    C = np.ascontiguousarray(C, dtype=np.float64).copy()
    A_cm = np.asfortranarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A_cm.shape
    n = B.shape[1]
    _k(lib.hplk_dgemm_update(m, n, k, ptr(A_cm), max(m, 1), ptr(B), max(n, 1), ptr(C),
                             max(n, 1), cfg), "hplk_dgemm_update")
    return C


def hplk_trsm(L, B):
    """L^{-1} B with L unit lower (device: unit-lower inverse + DMMA)."""
    L_cm = np.asfortranarray(L, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64).copy()
    k, n = B.shape
    _k(lib.hplk_trsm(k, n, ptr(L_cm), k, ptr(B), n), "hplk_trsm")
    return B


def hplk_panel_fact(Pn, nbmin: int = 16, leaf_variant: int = 0, leaf_cluster: int = 1,
                    leaf_ctas: int = 0):
    """Device panel LU of an m x nb panel with the chosen pivot-picking leaf
    (include/hpl_kernels.h). Returns (LU, ipiv, info)."""
    P_cm = np.array(Pn, dtype=np.float64, order="F", copy=True)
    m, nb = P_cm.shape
    ipiv = np.zeros(nb, dtype=np.int64)
    info = ctypes.c_int64(-1)
    st = lib.hplk_panel_fact(m, nb, ptr(P_cm), m, ptr(ipiv), nbmin, leaf_variant, leaf_cluster,
                             leaf_ctas, ctypes.byref(info))
    if st not in (0, -2):
        _k(st, "hplk_panel_fact")
    return np.ascontiguousarray(P_cm), ipiv, int(info.value)


def hplk_laswp(A, j0: int, ipiv, c0: int = 0, c1: int | None = None):
    """Device LASWP gather/scatter.  Returns (A_after, U) — U holds the block's
    final rows of columns [c0, c1); A's block rows in those columns are left
    as they were (hpl_factor overwrites them with the DTRSM result)."""
    A = np.ascontiguousarray(A, dtype=np.float64).copy()
    rows, cols = A.shape
    ipiv = np.ascontiguousarray(ipiv, dtype=np.int64)
    jb = len(ipiv)
    c1 = cols if c1 is None else c1
    U = np.zeros((jb, max(c1 - c0, 1)), dtype=np.float64)
    _k(lib.hplk_laswp(rows, cols, ptr(A), cols, j0, jb, ptr(ipiv), c0, c1, ptr(U),
                      U.shape[1]), "hplk_laswp")
    return A, U[:, : c1 - c0]


def hplk_rs_exchange(A, NB: int, P: int, j0: int, ipiv):
    """Device RS over P emulated process rows (rs_gather_peer + rs_scatter).
    Returns (A_after, U) like hplk_laswp (block rows of A left as they were)."""
    A = np.ascontiguousarray(A, dtype=np.float64).copy()
    rows, cols = A.shape
    ipiv = np.ascontiguousarray(ipiv, dtype=np.int64)
    jb = len(ipiv)
    U = np.zeros((jb, cols), dtype=np.float64)
    _k(lib.hplk_rs_exchange(rows, cols, ptr(A), cols, NB, P, j0, jb, ptr(ipiv), ptr(U), cols),
       "hplk_rs_exchange")
    return A, U


def hplk_back_solve(U, y, NB: int = 64):
    U = np.ascontiguousarray(U, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    N = U.shape[0]
    x = np.empty(N, dtype=np.float64)
    _k(lib.hplk_back_solve(N, NB, ptr(U), U.shape[1], ptr(y), ptr(x)), "hplk_back_solve")
    return x


def hplk_generate(seed: int, N: int, i0: int, rows: int, j0: int, cols: int):
    out = np.empty((rows, cols), dtype=np.float64)
    _k(lib.hplk_generate(seed, N, i0, rows, j0, cols, ptr(out)), "hplk_generate")
    return out


def hplk_residual(seed: int, N: int, x, want_rows: bool = False):
    """Device scaled residual of the seeded system for x (the hpl_residual
    kernels).  Returns (resid, out4) or, with want_rows, (resid, out4, rsum, asum)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out4 = np.zeros(4, dtype=np.float64)
    r = ctypes.c_double()
    rs = np.empty(N, dtype=np.float64) if want_rows else None
    as_ = np.empty(N, dtype=np.float64) if want_rows else None
    _k(lib.hplk_residual(seed, N, ptr(x), ptr(rs) if want_rows else None,
                         ptr(as_) if want_rows else None, ptr(out4), ctypes.byref(r)),
       "hplk_residual")
    return (float(r.value), out4, rs, as_) if want_rows else (float(r.value), out4)


def hplk_dgemm_bench(m: int, n: int, k: int, cfg: int = -1, reps: int = 5) -> np.ndarray:
    """Per-launch device times (ms) of the trailing DGEMM on resident operands."""
    ms = np.zeros(reps, dtype=np.float64)
    _k(lib.hplk_dgemm_bench(m, n, k, cfg, reps, ptr(ms)), "hplk_dgemm_bench")
    return ms


def hplk_dmma_peak(iters: int = 20000, blocks_per_sm: int = 2, warps: int = 8) -> float:
    """Measured FP64 tensor-pipe ceiling in TFLOP/s (register-resident DMMA chain)."""
    o = np.zeros(2, dtype=np.float64)
    _k(lib.hplk_dmma_peak(iters, blocks_per_sm, warps, ptr(o)), "hplk_dmma_peak")
    return o[1] / (o[0] * 1e-3) / 1e12


def hplk_panel_bench(m: int, nb: int = 512, nbmin: int = 16, leaf_ctas: int = 0,
                     reps: int = 3) -> np.ndarray:
    """Per-rep device time (ms) of the panel FACT of an m x nb panel."""
    ms = np.zeros(reps, dtype=np.float64)
    _k(lib.hplk_panel_bench(m, nb, nbmin, leaf_ctas, reps, ptr(ms)), "hplk_panel_bench")
    return ms
