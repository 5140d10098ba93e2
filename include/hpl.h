/*
 * hpl.h — C ABI of libhpl.so, the B200-native HPL hot path.
 *
 * The library solves A x = b for a dense, seeded, random FP64 system by
 * blocked right-looking LU with partial pivoting on a 2D block-cyclic P x Q
 * process grid, one process per B200 ("let every MPI process
 * manage one and only one GPU device").  The whole matrix stays resident in
 * HBM; every phase — panel FACT, LBCAST, RS/LASWP, the DTRSM of
 * the U block row and the trailing DGEMM with look-ahead
 * — runs as this library's own sm_100a kernels and NCCL calls; the host only
 * enqueues work.  Definitions of the phases: SPEC.md glossary l.543–552;
 * operation order: SURVEY.md §3.4 and DESIGN.md.
 *
 * Conventions common to every entry point
 *  - Matrix: the N x (N+1) augmented matrix [A | b] (b is global column N, so
 *    row interchanges reach b for free).  Entry (i, j) is
 *    g(seed, j*N + i) with g the SplitMix64-based generator of DESIGN.md
 *    reading A6: uniform on the 2^-53 grid in [-0.5, 0.5).
 *  - Distribution: NB x NB blocks, block (I, J) on process (I mod P, J mod Q);
 *    rank = p + q*P (column-major).  Local storage is ROW-major
 *    with a padded leading dimension.
 *  - Pivots: LAPACK 0-based global row indices (ipiv[k] = row exchanged with
 *    row k at step k); ties -> smallest global row (DESIGN reading A2).
 *  - Threading: a context is not thread-safe, but different contexts may be
 *    driven from different host threads at once (the library keeps no
 *    process-wide mutable state); the loopback grid (hpl_init_loopback)
 *    needs exactly that.  On a multi-rank context every call is collective
 *    over all P*Q ranks and must be made in the same order.
 *  - Call order: init -> factor -> solve -> residual; regenerate / load_local
 *    reset to "initialised".  Out-of-order calls return HPL_ERR_STATE.
 *  - Errors never abort the process: a status is returned and
 *    hpl_last_error() describes it.  CUDA and NCCL failures map to
 *    HPL_ERR_CUDA / HPL_ERR_NCCL; the context should then be freed.
 *  - Failure detection: every device-side wait on another rank (RS and FACT
 *    barriers, the pivot exchange, LBCAST flags, collectives) is bounded by
 *    the peer timeout (option peer_timeout_ms; 60 s, 20 s in a loopback).  A
 *    rank that dies or does not enter a collective call makes its peers'
 *    call return HPL_ERR_PEER instead of hanging; the
 *    context is then broken and must be freed.
 *  - Argument limits (HPL_ERR_ARG, before any allocation): N >= 1,
 *    1 <= NB <= N, P, Q >= 1 and the implementation
 *    limits of DESIGN.md reading A18: NB even and <= 1024, N < 2^31, P <= 8,
 *    Q <= 32, P*Q <= 32.
 *  - Ownership: the library owns all device memory, streams, events and NCCL
 *    communicators (freed by hpl_free).  Host pointers are caller-owned and
 *    only read/written during the call.
 */
#ifndef HPL_B200_H
#define HPL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hpl_ctx hpl_ctx;

typedef enum {
    HPL_OK = 0,
    HPL_ERR_ARG = 1,      /* invalid argument; nothing allocated */
    HPL_ERR_STATE = 2,    /* call out of order */
    HPL_ERR_OOM = 3,      /* device allocation failed (only at init) */
    HPL_ERR_CUDA = 4,     /* CUDA runtime/driver error */
    HPL_ERR_NCCL = 5,     /* NCCL error */
    HPL_ERR_SINGULAR = 6, /* exact zero pivot; see hpl_singular_column */
    HPL_ERR_PEER = 7      /* a peer-memory wait timed out: a peer rank failed or is absent */
} hpl_status;

/* Single-process context on the current CUDA device.  P*Q must be 1.
 * N >= 1, 1 <= NB <= N (HPL_ERR_ARG otherwise, before any
 * allocation).  Allocates the local (N x (N+1)) matrix plus workspaces and
 * fills it from `seed` with the device generator. */
hpl_status hpl_init(int64_t N, int32_t NB, int32_t P, int32_t Q, uint64_t seed,
                    hpl_ctx **out);

/* Multi-process context (collective over nranks = P*Q processes, one per GPU).
 * rank = p + q*P; nccl_unique_id points to the 128-byte ncclUniqueId that
 * rank 0 created and every rank received out of band (e.g. through
 * torch.distributed); device is the CUDA ordinal this rank drives.
 * All ranks must be on one node with peer access (NVLink/NVSwitch): the
 * context exchanges CUDA IPC handles (over NCCL) so that the P processes of a
 * process column map each other's local matrix, pivot-exchange area and RS
 * flags, and the Q processes of a process row map each other's panel buffers
 * and LBCAST flags.  A failed IPC
 * open returns HPL_ERR_CUDA. */
hpl_status hpl_init_dist(int64_t N, int32_t NB, int32_t P, int32_t Q, uint64_t seed,
                         int32_t rank, int32_t nranks, const void *nccl_unique_id,
                         int32_t device, hpl_ctx **out);

/* Single-device P x Q loopback ("ranks are concurrent workers
 * in one process"): creates the P*Q rank contexts of one grid on CUDA device
 * `device` of THIS process, out[r] = rank r (r = p + q*P).  They run exactly
 * the multi-GPU data path — peer-memory RS, pivot exchange, LBCAST flags and
 * collectives, with the siblings' device pointers in place of IPC mappings —
 * so one GPU checks it against the oracle.  Each collective call must be made
 * on every rank concurrently, one host thread per rank.  Because the ranks'
 * kernels wait on each other, the process must run with
 * CUDA_MODULE_LOADING=EAGER and CUDA_DEVICE_MAX_CONNECTIONS >= 3*P*Q set
 * before CUDA initialises (HPL_ERR_STATE otherwise, when P*Q > 1); each
 * rank's cooperative leaf is capped at SMs/(P*Q) CTAs so all fit at once.
 * On failure the already-created contexts are still returned in out (free
 * them).  Free every rank only after all ranks' calls have returned. */
hpl_status hpl_init_loopback(int64_t N, int32_t NB, int32_t P, int32_t Q, uint64_t seed,
                             int32_t device, hpl_ctx **out);

/* Writes a fresh ncclUniqueId (128 bytes) into id_out (rank 0 only). */
hpl_status hpl_get_unique_id(void *id_out);

/* In-place LU with partial pivoting of the local [A | b] (collective).
 * Blocks until the factorization is complete on this rank.  Returns
 * HPL_ERR_SINGULAR if an exact zero pivot occurred. */
hpl_status hpl_factor(hpl_ctx *ctx);

/* Back substitution U x = y (y = the eliminated column N).  x is replicated on
 * every rank; if x_host is non-NULL the N doubles are copied there. */
hpl_status hpl_solve(hpl_ctx *ctx, double *x_host);

/* HPL scaled residual ||A0 x - b0||_inf / (eps (||A0||_inf ||x||_inf +
 * ||b0||_inf) N), eps = 2^-53 (reading A4), regenerating A0 and b0 from the
 * seed on the fly (the factors are not touched).  Requires hpl_solve.  A
 * non-finite x or norm gives +inf (a failed solve never passes "< 16").
 * After hpl_load_local the factored system is not the seeded one:
 * HPL_ERR_STATE. */
hpl_status hpl_residual(hpl_ctx *ctx, double *resid);

/* Refill the local matrix from the seed (returns to the initialised state). */
hpl_status hpl_regenerate(hpl_ctx *ctx);

/* Load this rank's local block of [A | b] from a HOST buffer laid out exactly
 * like the device copy: local_rows x local_cols row-major with leading
 * dimension ld (>= local_cols); see hpl_local_shape.  Used by end-to-end
 * timing and tests with hand-made systems.  Returns to "initialised". */
hpl_status hpl_load_local(hpl_ctx *ctx, const double *host, int64_t ld);

/* hpl_load_local + hpl_factor with the host->device copy overlapped with
 * the factorization (contexts with >= 4 panel buffers, decided at init from
 * free memory and the same on every rank; otherwise the two calls).  Each
 * rank passes its own local block.  The local block is copied in column chunks on a copy stream and
 * the updates of the first iterations run per chunk behind the arrivals
 * (DESIGN.md §5 "Pipelined start"), so most of the copy hides behind the
 * DGEMMs; the arithmetic per element is unchanged, the result is bitwise that
 * of the two calls.  `host` should be page-locked (hpl_pin_host) for the copy
 * to be asynchronous; it is read during the call only.  Collective; returns
 * like hpl_factor; afterwards the context holds a loaded system
 * (hpl_residual: HPL_ERR_STATE). */
hpl_status hpl_load_factor(hpl_ctx *ctx, const double *host, int64_t ld);

/* Local extents of [A | b] on this rank (rows, cols incl. b when owned). */
hpl_status hpl_local_shape(const hpl_ctx *ctx, int64_t *rows, int64_t *cols);

void hpl_free(hpl_ctx *ctx);
const char *hpl_last_error(const hpl_ctx *ctx);
int64_t hpl_singular_column(const hpl_ctx *ctx); /* -1 if none */

/* ---- test / measurement hooks ---- */
/* Global pivots of the last factorization, N entries (identical on all ranks). */
hpl_status hpl_get_ipiv(const hpl_ctx *ctx, int64_t *ipiv_host);
/* Copy the local [A | b] block (after factor: L\U in HPL row order and y) to
 * host, row-major with leading dimension ld >= local cols. */
hpl_status hpl_get_local(const hpl_ctx *ctx, double *host, int64_t ld);
/* Per-iteration phase times in ms, 6 doubles per iteration:
 * [fact, la_update, rest_update, laswp, trsm, dgemm_rest]; returns the number
 * of iterations written (<= cap). */
int64_t hpl_get_timeline(const hpl_ctx *ctx, double *t, int64_t cap);
/* Breakdown of the timeline's fact phase, 3 doubles per iteration j (ms):
 * [wait for the trailing RS + DTRSM of iteration j before FACT(j+1),
 *  FACT(j+1) proper on the owner process column (0 elsewhere: pack, factor,
 *  write back, incl. the P>1 pivot exchange), LBCAST(j+1) + pivot plan +
 *  L11^{-1}].  Zeros for the last iteration.  Needs hpl_set_timing(ctx, 1)
 * before hpl_factor; returns the number of iterations written (<= cap). */
int64_t hpl_get_fact_detail(const hpl_ctx *ctx, double *t, int64_t cap);
/* Enable per-phase CUDA events (adds a little host work per iteration). */
hpl_status hpl_set_timing(hpl_ctx *ctx, int32_t enable);
/* Tuning / A-B knobs (none changes the pivots; each is tested against the
 * oracle or bitwise against the default in tests/):
 *   lookahead 0|1 (1)      look-ahead depth 1 on high-priority streams
 *   split <pct> (0)        split update, right-section share
 *   rs_peer 0|1 (1)        P>1 RS as a peer-memory row gather; 0 = collective
 *                          variant (U all-reduced, W broadcast over the column)
 *   lb_peer 0|1 (1)        Q>1 LBCAST as copy-engine pulls; 0 = broadcast collective
 *   coll_nccl 0|1 (0)      multi-process: the collectives (replicated top block,
 *                          back-solve sums/broadcasts, residual norms, rs_peer=0 /
 *                          lb_peer=0 variants) over NCCL instead of peer memory
 *                          (NCCL waits are not bounded by peer_timeout_ms)
 *   peer_timeout_ms <ms>   bound of every device-side wait on a peer (60000)
 *   nbmin <1..16> (16)     recursion base width of the panel FACT
 *   fact_gather <rows> (65536), fact_gather_ms <ms> (8)  P>1: a panel with at
 *                          most this many global rows whose per-GPU trailing
 *                          update is estimated below fact_gather_ms (FACT on the
 *                          critical path) is factored whole on every GPU of the
 *                          process column (gathered over peer memory) instead of
 *                          by the distributed leaf; fact_gather 0 = never
 *   leaf_cluster 0|1 (1)   small panels (<= 16 x 1664 rows) factored by one 16-CTA
 *                          cluster with the leaf in shared memory
 *   leaf_variant 0|1|2 (0) P=1 FACT leaf: right-looking / left-looking / Crout
 *                          (bitwise-equal results)
 *   leaf_few_ctas <n> (8), leaf_hide_ms <ms> (15), leaf_warp <n> (0), leaf_ctas <n>
 *                          leaf grid policy: while the concurrent trailing DGEMM
 *                          is estimated longer than leaf_hide_ms the leaf runs on
 *                          leaf_few_ctas CTAs (or leaf_warp one-warp CTAs), else
 *                          on every SM; leaf_ctas fixes the grid
 *   gemm_cfg -1|0|1|2 (-1) DGEMM tile config (128x64, 128x128, 64x64 = default)
 * Every knob is per context.  Unknown names return HPL_ERR_ARG.  On a multi-process context every rank
 * must set the same options before the same hpl_factor (the schedule decides
 * which collectives and peer-memory barriers are issued). */
hpl_status hpl_set_option(hpl_ctx *ctx, const char *name, int64_t value);
/* Number of this library's kernel launches in the last hpl_factor + hpl_solve. */
int64_t hpl_launch_count(const hpl_ctx *ctx);
/* Device-timed (CUDA events on the library's streams) results of the last
 * factor/solve: out6 = {factor_ms, solve_ms, trailing-DGEMM launches,
 * trailing-DGEMM ms (sum of per-launch event pairs), trailing-DGEMM flop,
 * kernel launches}.  The DGEMM entries are filled only with hpl_set_timing(1). */
hpl_status hpl_last_timing(const hpl_ctx *ctx, double *out6);

/* Per-phase totals of the last hpl_factor / hpl_solve (CUDA events; the
 * factor entries need hpl_set_timing(1)), for the roofline of every
 * non-DGEMM kernel: out10 = {rest LASWP/RS ms, its algorithmic bytes
 * (2 x 8 x (jb + displaced rows) x rest columns per iteration: each moved
 * row read once and written once), rest DTRSM ms, its flop (jb^2 x rest
 * columns per iteration), FACT ms (owner column, summed over panels), solve
 * ms, the solve's algorithmic bytes (this rank's part of the upper triangle
 * of U, read once), trailing-DGEMM ms, and for hpl_load_factor: ms from the
 * factorization's start until the last column chunk landed, bytes copied,
 * ms until the pipelined start's iterations were done everywhere, their
 * number (0, 0, 0, 0 otherwise)} — 12 doubles. */
hpl_status hpl_phase_stats(const hpl_ctx *ctx, double *out10);

/* Debug hook: out = {group barrier counters (world, row, column, column-tr),
 * this rank's 4 x 32 group flag words (arrivals received per group and
 * member), the abort word and its detail} — 4 + 128 + 2 entries (cap must
 * be at least that).  For diagnosing a peer timeout. */
hpl_status hpl_debug_state(const hpl_ctx *ctx, uint64_t *out, int64_t cap);

/* Host-only bookkeeping of the P > 1 panel FACT of panel j on process row
 * myrow (DESIGN.md §6 "Gathered panel FACT"):
 * out5 = {mode (-1: P = 1, 0: distributed leaf, 1: gathered — a function of
 * the global sizes only, identical on every process row), global rows of the
 * panel N - j*NB, first local L row, number of local L rows, leading
 * dimension of the packed [T; L] panel}.  gather_rows / gather_ms as the
 * fact_gather / fact_gather_ms options.  HPL_ERR_ARG on invalid arguments. */
hpl_status hpl_plan_fact(int64_t N, int32_t NB, int32_t P, int32_t Q, int32_t myrow, int64_t j,
                         int64_t gather_rows, double gather_ms, int64_t *out5);
/* Host-only planning of iteration j for process (myrow, mycol) of a P x Q
 * grid (no GPU work; the factor loop uses the same bookkeeping):
 * out8 = {first active local row, first trailing local column, look-ahead
 * column range [b, e) (empty unless this process owns panel j+1), rest
 * column range [b, e), local column of panel j on its owner (-1 elsewhere),
 * jb}.  2D block-cyclic map of SPEC.md l.30–57. */
hpl_status hpl_plan_iteration(int64_t N, int32_t NB, int32_t P, int32_t Q, int32_t myrow,
                              int32_t mycol, int64_t j, int64_t *out8);
/* Page-lock (pin = 1) or release (pin = 0) a caller-owned host buffer so
 * hpl_load_local / hpl_solve copies run at full DMA speed. */
hpl_status hpl_pin_host(void *p, int64_t bytes, int32_t pin);

#ifdef __cplusplus
}
#endif
#endif /* HPL_B200_H */
