// hpl_internal.cuh — shared declarations of libhpl.so's kernels and launchers.
// Product code only; nothing here is shared with oracle/ (see DESIGN.md).
//
// Every knob lives in the caller's context (FactWork, the dgemm cfg
// argument): there is no process-wide mutable state, so several contexts can
// drive the library from several host threads at once (the single-device
// P x Q loopback).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>

namespace hpl {

// Number of this library's kernel launches issued by the calling host thread
// (each rank of a loopback grid runs on its own thread; reported as
// gpu_launches).
extern thread_local int64_t t_launches;
inline void count_launch(int64_t n = 1) { t_launches += n; }

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- bounded peer waits
// Every spin on a flag another rank (or another CTA) writes is bounded: it
// gives up when this context's abort word is set, or sets it (with a site
// code) once timeout_ns of %globaltimer have passed.  A dead or absent peer
// therefore ends hpl_factor / hpl_solve / hpl_residual with HPL_ERR_PEER
// instead of spinning forever (a deadlock surfaces as
// an error).  After an abort every later wait of the context returns at
// once, the kernels finish on garbage and the context must be freed.
struct SpinCtl {
    unsigned long long *abort;      // device word: 0 = running, else the first failing site
    unsigned long long timeout_ns;
};
enum SpinSite : unsigned {
    SITE_GRID_BARRIER = 1, SITE_DIST_PEER = 2, SITE_DIST_WIN = 3, SITE_RS_BARRIER = 4,
    SITE_FLAG = 5, SITE_GROUP_BARRIER = 6
};

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ bool spin_aborted(const SpinCtl &sc)
{
    return *reinterpret_cast<volatile const unsigned long long *>(sc.abort) != 0ull;
}
// Record the first abandoned wait: abort[0] = site code (low 4 bits: the
// SpinSite; above them a site-specific detail such as the group and member
// waited for), abort[1] = expected value << 32 | value seen (low 32 bits).
__device__ __forceinline__ void spin_record(const SpinCtl &sc, unsigned long long code,
                                            unsigned long long want, unsigned long long seen)
{
    if (atomicCAS(sc.abort, 0ull, code) == 0ull)
        sc.abort[1] = (want << 32) | (seen & 0xffffffffull);
}
// Wait until *p >= v (system-scope acquire).  false: abandoned (abort/timeout).
__device__ __forceinline__ bool spin_geq_sys(const unsigned long long *p, unsigned long long v,
                                             const SpinCtl &sc, unsigned long long site)
{
    if (ld_acquire_sys(p) >= v) return true;
    const unsigned long long t0 = gtimer();
    for (unsigned n = 1;; ++n) {
        if (ld_acquire_sys(p) >= v) return true;
        if ((n & 15u) == 0) {
            if (spin_aborted(sc)) return false;
            if (gtimer() - t0 > sc.timeout_ns) {
                spin_record(sc, site, v, ld_acquire_sys(p));
                return false;
            }
        }
        __nanosleep(64);
    }
}
// Same at GPU scope (flags written by other CTAs of this GPU).
__device__ __forceinline__ bool spin_geq_gpu(const unsigned long long *p, unsigned long long v,
                                             const SpinCtl &sc, unsigned long long site)
{
    if (ld_acquire_gpu(p) >= v) return true;
    const unsigned long long t0 = gtimer();
    for (unsigned n = 1;; ++n) {
        if (ld_acquire_gpu(p) >= v) return true;
        if ((n & 63u) == 0) {
            if (spin_aborted(sc)) return false;
            if (gtimer() - t0 > sc.timeout_ns) {
                spin_record(sc, site, v, ld_acquire_gpu(p));
                return false;
            }
        }
    }
}
#endif

// ---------------------------------------------------------------- generator
// Fill local block: rows [0, lrows) x cols [0, lcols) of the row-major local
// matrix (ld) with entries of the global N x (N+1) system, local->global via
// the block-cyclic map (NB, P, Q, myrow, mycol).
cudaError_t gen_local(cudaStream_t st, uint64_t seed, int64_t N, int NB, int P, int Q,
                      int myrow, int mycol, int64_t lrows, int64_t lcols, double *A, int64_t ld);
// Fill an explicit global window (tests).
cudaError_t gen_window(cudaStream_t st, uint64_t seed, int64_t N, int64_t i0, int64_t rows,
                       int64_t j0, int64_t cols, double *out, int64_t ld);

// ---------------------------------------------------------------- copies
// dst (col-major, ldd) <- src (row-major, lds): rows x cols.
cudaError_t rm_to_cm(cudaStream_t st, int64_t rows, int64_t cols, const double *src, int64_t lds,
                     double *dst, int64_t ldd);
// dst (row-major, ldd) <- src (col-major, lds): rows x cols.
cudaError_t cm_to_rm(cudaStream_t st, int64_t rows, int64_t cols, const double *src, int64_t lds,
                     double *dst, int64_t ldd);

// ---------------------------------------------------------------- DGEMM
enum GemmMode { GEMM_UPDATE = 0, GEMM_ASSIGN = 1 };
// C (m x n row-major ldc)  -=  A (m x k col-major lda) * B (k x n row-major ldb)   [UPDATE]
// C                         =  A * B                                              [ASSIGN]
// a_lower: A is lower triangular (A[i][p] = 0 for p > i): k-chunks above the
// diagonal of each m-tile are skipped.  A and B must be 16-byte aligned with
// even lda/ldb (TMA); C may be anywhere.  C2 (ASSIGN only, 16B aligned, even
// ldc2): the epilogue stores the result there as well.  cfg: tile config
// (0: 128x64, 1: 128x128, 2: 64x64 = DGEMM_DEFAULT_CFG; -1 = default).
// slot selects the param-space offset of the kernel's tensor maps: launches
// that may run concurrently must use different slots (see kernels_gemm.cu
// ParamPad); the driver picks the slot from the stream.
constexpr int DGEMM_DEFAULT_CFG = 2;
enum GemmSlot { SLOT_TRAIL = 0, SLOT_LOOKAHEAD = 1, SLOT_FACT = 2, SLOT_RS = 3 };
cudaError_t dgemm(cudaStream_t st, int mode, bool a_lower, int64_t m, int64_t n, int64_t k,
                  const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                  int64_t ldc, int cfg = -1, double *C2 = nullptr, int64_t ldc2 = 0,
                  int slot = SLOT_TRAIL);

// ---------------------------------------------------------------- TRSM helpers
// In-place B (k x ncols, col-major ldb) <- L^{-1} B, L unit lower (col-major ldl),
// one CTA per column of B.  If identity_init, B is first set to I (k x k) —
// then B = L^{-1}.
cudaError_t trsm_cols(cudaStream_t st, int64_t k, int64_t ncols, const double *L, int64_t ldl,
                      double *B, int64_t ldb, bool identity_init);

// ---------------------------------------------------------------- panel FACT
// Per-context FACT workspace and leaf policy (formerly process-wide knobs).
struct FactWork {
    double *cand;        // candidate records (2 parity buffers)
    unsigned *bar;       // grid barrier words (count, generation) + winner flag
    int64_t *info;       // first singular global column; all-ones (== -1) if none
    double *win;         // P > 1: winning pivot record (global row + full panel row)
    double *tsnap;       // P > 1: snapshot of the replicated top row kc
    unsigned long long *abort;   // SpinCtl abort word of the owning context
    unsigned long long timeout_ns;
    int max_ctas;        // hard cap of every leaf grid (loopback: SMs / ranks)
    int num_sms;
    // leaf policy
    int leaf_max_ctas = 0;       // 0 = all SMs (up to max_ctas)
    int leaf_rows_per_cta = 512;
    int leaf_warp_ctas = 0;      // > 0: one-warp CTAs (co-resident with the DGEMM), at most this many
    int leaf_variant = 0;        // 0 right-looking, 1 left-looking, 2 Crout
    int leaf_cluster = 1;        // one-cluster shared-memory leaf for small panels
    int gemm_cfg = -1;           // DGEMM tile config of the recursion's updates
    int plain_launch = 0;        // loopback: leaf grids by a plain launch (kernels_fact.cu launch_grid)
    SpinCtl spin() const { return SpinCtl{abort, timeout_ns}; }
};

// P > 1 panel FACT: the P processes of the panel's process column exchange
// pivot candidates (value, global row, full panel row) through peer memory
// (CUDA IPC over NVLink, or plain pointers in the loopback) inside the leaf.
constexpr int MAX_P = 8;
struct DistExchange {
    double *rec[MAX_P];                 // record area on each peer (index = process row)
    unsigned long long *flag[MAX_P];    // flag area on each peer
    double *my_rec;                     // = rec[myrow]
    unsigned long long *my_flag;        // = flag[myrow]
    int P, myrow, recd;                 // recd = doubles per record (2 + NB)
};
// Panel rows [0, jbp) are the replicated top block T (global rows j0..j0+jbp);
// rows jbp.. are this process row's other active rows, the first being local
// row lrL0 (global row via the block-cyclic map with NB, P, myrow).
struct DistPanel {
    long long j0, lrL0;
    int jbp, is_prow, NB, P, myrow;
};
struct DistFact {
    DistPanel dp;
    DistExchange ex;
    unsigned long long *seq;            // host counter, advanced once per panel column
};
cudaError_t fact_work_alloc(FactWork *w);
// Leaf grid size: min(max_ctas (0 = #SMs), ceil(rows / rows_per_cta)).  Fewer
// CTAs leave more of each SM to the concurrent trailing DGEMM.
void fact_set_leaf_ctas(FactWork *w, int max_ctas, int rows_per_cta);
// Gathered panel FACT (P > 1, small panels): every process of the column
// builds the combined panel (row c = global row j0 + c) from the packed
// panels of all P processes (peer memory), factors it with the one-GPU FACT
// (bitwise the same arithmetic as the distributed leaf), and extracts its own
// rows.  panel[p] / ld[p] / lrL0[p]: process row p's packed panel of this panel.
struct FactPeers {
    const double *panel[MAX_P];
    long long ld[MAX_P];
    long long lrL0[MAX_P];
    int myrow;
};
cudaError_t fact_gather(cudaStream_t st, int64_t rows, int64_t jb, int64_t j0, int NB, int P,
                        const FactPeers &fp, double *Cp, int64_t ldc);
cudaError_t fact_extract(cudaStream_t st, int64_t mine, int64_t jb, int64_t j0, int NB, int P,
                         int myrow, int64_t lrL0, const double *Cp, int64_t ldc, double *Pn,
                         int64_t ldp);
void fact_work_free(FactWork *w);
// Recursive right-looking panel LU (NDIV=2, leaf nbmin) of P (m x nb col-major ldp).
// ipiv receives panel-relative pivots (device, int64).  Uses scratch for the
// transposed U block of the recursion GEMMs (>= nb*nb doubles).  A zero pivot
// at panel column k records min(goff + k) in w->info.
cudaError_t panel_fact(cudaStream_t st, int64_t m, int64_t nb, double *P, int64_t ldp,
                       int64_t *ipiv_dev, int nbmin, FactWork *w, double *scratch, int64_t goff,
                       DistFact *dist = nullptr);

// ---------------------------------------------------------------- LASWP
// From panel-relative pivots (jb entries; positions r0+k <-> r0+ipiv_rel[k])
// build: src[k] (row whose content ends in row r0+k, k<jb), and ndisp
// displaced (dst, src) row pairs (dst >= r0+jb).  Also writes global pivots
// gpiv[k] = ipiv_rel[k] + goff.  Rows are < nrows; a pivot outside
// [r0+k, nrows) (only after an aborted FACT) is taken as no interchange.
// All device arrays.
cudaError_t pivot_plan(cudaStream_t st, int64_t jb, int64_t r0, const int64_t *ipiv_rel,
                       int64_t goff, int64_t nrows, int64_t *gpiv, int64_t *src, int64_t *disp,
                       int *ndisp);
// Gather U[k][c] = A[src[k]][c0+c] and scatter A[disp_dst][c] = A[disp_src][c]
// for columns [c0, c1) of the row-major A.
cudaError_t laswp_gather_scatter(cudaStream_t st, int64_t jb, const int64_t *src,
                                 const int64_t *disp, const int *ndisp, double *A, int64_t lda,
                                 int64_t c0, int64_t c1, double *U, int64_t ldu);

// P > 1 row swaps (RS): pack the rows of U this process row owns (zeros
// elsewhere; summed over the process column by the caller), and scatter the
// displaced rows from W = the original block row (broadcast from its owner).
// src / disp hold GLOBAL rows; NB, P, myrow give the global->local row map.
cudaError_t rs_pack(cudaStream_t st, int64_t jb, const int64_t *src, const double *A, int64_t lda,
                    int64_t c0, int64_t c1, double *U, int64_t ldu, int NB, int P, int myrow);
cudaError_t rs_scatter(cudaStream_t st, const int64_t *disp, const int *ndisp, const double *W,
                       int64_t ldw, int64_t j0, double *A, int64_t lda, int64_t c0, int64_t c1,
                       int NB, int P, int myrow);

// P > 1 RS over peer memory: A[p] = process row p's local A (IPC-mapped; own
// A at myrow), flag[p] = its barrier flag area (RS_SLOTS x MAX_P u64),
// my_flag = this process's.  Process rows of one process column share lda.
constexpr int RS_SLOTS = 8;
struct RsPeers {
    const double *A[MAX_P];
    unsigned long long *flag[MAX_P];
    unsigned long long *my_flag;
    int P, myrow;
};
// Flag barrier over the process column at `slot` (monotonic value): one
// one-warp kernel; every later kernel on st sees the peers' earlier writes.
cudaError_t rs_barrier(cudaStream_t st, const RsPeers &pr, int slot, unsigned long long value,
                       const SpinCtl &sc);
// Phase 1 of the peer-memory RS for local columns [c0, c1): U[k] = global row
// src[k] read from its owner; W[s - j0] = original block row s (from the
// owner of block row j0) for every displaced pair (d, s) whose d this process owns.
cudaError_t rs_gather_peer(cudaStream_t st, int64_t jb, const int64_t *src, const int64_t *disp,
                           const int *ndisp, const RsPeers &pr, int64_t lda, int64_t c0,
                           int64_t c1, double *U, int64_t ldu, double *W, int64_t ldw, int64_t j0,
                           int NB);

// One flag step over peer memory (LBCAST): publish sv to each sig[i] (i <
// nsig), then wait until every *wt[i] >= wv (i < nwait).  One one-warp kernel.
struct FlagOp {
    unsigned long long *sig[32];
    const unsigned long long *wt[32];
    int nsig, nwait;
    unsigned long long sv, wv;
};
cudaError_t flag_op(cudaStream_t st, const FlagOp &op, const SpinCtl &sc);

// ---------------------------------------------------------------- peer collectives
// Collectives over a group of ranks (world / process row / process column)
// through peer memory, for the exchanges that are not the hot-path RS /
// LBCAST / pivot search: the replicated top block of the P > 1 FACT, the
// back-solve reductions and broadcasts, the residual norms, the singular
// column.  Each rank owns a CommBlock (device memory, IPC-mapped by its peers
// or a plain pointer in the loopback); a collective stages this rank's data
// in its own block, passes a flag barrier, reads every member's stage in a
// fixed member order (the same result bits on every rank), and passes a
// second barrier before the stage is reused.
constexpr int MAX_GROUP = 32;
constexpr int N_GROUPS = 4;                       // world, row, column, column (trailing stream)
constexpr int64_t STAGE_DOUBLES = int64_t(1) << 19;   // 4 MB per group
struct CommBlock {
    unsigned long long flag[N_GROUPS][MAX_GROUP];   // barrier arrival words [group][member]
    double stage[N_GROUPS][STAGE_DOUBLES];
};
struct GroupDev {
    CommBlock *blk[MAX_GROUP];    // member m's block (own block at index me)
    int size, me, gid;
};
enum CollOp { COLL_SUM = 0, COLL_MAX = 1, COLL_MIN_U64 = 2 };
cudaError_t group_barrier(cudaStream_t st, const GroupDev &g, unsigned long long value,
                          const SpinCtl &sc);
// Device-to-device 2D copy (rows x width bytes) and an 8-byte store, done by
// SMs instead of the copy engine: the loopback's copies (hpl_comm.cu d2d).
cudaError_t copy2d_sm(cudaStream_t st, void *dst, int64_t dpitch, const void *src, int64_t spitch,
                      int64_t width, int64_t rows);
cudaError_t fill_u64(cudaStream_t st, unsigned long long *p, unsigned long long v);
// out[i] = op over members m = 0..size-1 (in order) of member m's stage[gid][i].
cudaError_t group_reduce(cudaStream_t st, const GroupDev &g, int op, int64_t n, void *out);

// ---------------------------------------------------------------- solve / residual
// Single-matrix back solve (y = column N of U's rows): hplk_back_solve.
cudaError_t back_solve(cudaStream_t st, int64_t N, int NB, const double *U, int64_t ldu,
                       const double *y, int64_t ystride, double *x, double *tbuf);
// partial[s][r] (s < S, nb apart): the sum over the s-th share of the local
// NB-blocks of Urows[r][c] x[gcol(c)], lc_lo <= c < lc_hi, minus Urows[r][lcy]
// in share 0 when lcy >= 0.  S <= 16 (bs_splits suggests one); partial holds S * nb doubles.
int bs_splits(int nb, int64_t lc_lo, int64_t lc_hi, int NB);
cudaError_t bs_partial(cudaStream_t st, int nb, const double *Urows, int64_t ldu, int64_t lc_lo,
                       int64_t lc_hi, int NB, int Q, int mycol, const double *x, int64_t lcy,
                       double *partial, int S);
// xb = U_bb^{-1} (-sum_s partial[s] - U_near x_near): nnear > 0 folds the
// near sums (the next nnear columns of the block's rows times xnear) into the
// solve; only when bs_diag_folds_near(nb) (the cluster solve is available).
cudaError_t bs_diag(cudaStream_t st, int nb, const double *Ubb, int64_t ldu,
                    const double *partial, int S, double *xb, int nnear = 0,
                    const double *xnear = nullptr);
bool bs_diag_folds_near(int nb);
// Residual of the seeded system: per-rank partial sums (local rows x local
// columns), then (after the caller's all-reduce over the process row) the
// norms into out4 = {rinf, anorm, xnorm, bnorm} (max over local rows; a
// non-finite value anywhere makes the corresponding entry +inf).
cudaError_t residual_partial(cudaStream_t st, uint64_t seed, int64_t N, int NB, int P, int myrow,
                             int64_t mloc, int Q, int mycol, int64_t lcols, const double *x,
                             double *r, double *a);
cudaError_t residual_finalize(cudaStream_t st, uint64_t seed, int64_t N, int NB, int P, int myrow,
                              int64_t mloc, const double *r, const double *a, const double *x,
                              double *out4);

// HPL's scaled residual from out4 = {||r||, ||A0||, ||x||, ||b0||} (SPEC.md
// l.383-391, eps = 2^-53, reading A4); a non-finite part gives +inf.
inline double scaled_residual(const double *h, int64_t N)
{
    for (int k = 0; k < 4; ++k)
        if (!(h[k] - h[k] == 0.0)) return __builtin_inf();   // inf or NaN
    const double r = h[0] / (0x1p-53 * (h[1] * h[2] + h[3]) * (double)N);
    return r == r ? r : __builtin_inf();
}

// Set every kernel attribute (dynamic shared memory sizes, cluster
// permissions) once per process, before any rank runs: the first
// cudaFuncSetAttribute of a kernel must not happen inside one loopback rank
// while others' kernels already wait on it (hpl_comm.cu alloc_ctx).
cudaError_t dgemm_prepare();
cudaError_t fact_prepare();
cudaError_t solve_prepare();

// FP64 tensor-pipe ceiling: register-resident DMMA chain on every SM.
cudaError_t dmma_peak(int iters, int blocks_per_sm, int warps, double *ms, double *flop);

}  // namespace hpl

#define HPL_CUDA_TRY(expr)                              \
    do {                                                \
        cudaError_t _e = (expr);                        \
        if (_e != cudaSuccess) return _e;               \
    } while (0)
