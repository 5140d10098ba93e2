// kernels_swap.cu — LASWP gather/scatter around the pivot exchange
// ("a GPU kernel to gather the rows to
// be communicated ... and a GPU kernel to scatter the received rows back").
//
// The jb sequential swaps (r0+k) <-> ipiv[k] of one panel are first turned
// into a plan: src[k] = the row whose content ends in row r0+k, and the list
// of rows below the block that receive a row of the block (every swap has a
// block row as its first element, so content that reaches the block never
// leaves it again, and a row below the block can only receive an ORIGINAL
// block row).  With the plan, one pass over the trailing columns moves each
// row once: the block's final rows are gathered into the U buffer (the DTRSM
// then writes L11^{-1} U back into block row r0) and the displaced rows are
// scattered — coalesced 16-byte row copies, HBM-bound.
#include "hpl_internal.cuh"

namespace hpl {

namespace {

constexpr int HSLOTS = 2048;  // open-addressing table for rows below the block (jb <= 1024)

// A pivot outside [r0 + k, nrows) cannot come from a FACT that completed; it
// only appears after a peer timeout abandoned the leaf (hpl_internal.cuh
// SpinCtl).  It is treated as "no interchange" so no later kernel indexes
// outside the matrix; the context reports HPL_ERR_PEER.
__global__ void pivot_plan_kernel(int jb, long long r0, const int64_t *__restrict__ ipiv_rel,
                                  long long goff, long long nrows, int64_t *gpiv, int64_t *src,
                                  int64_t *disp, int *ndisp)
{
    __shared__ long long keys[HSLOTS];
    __shared__ long long vals[HSLOTS];
    __shared__ long long cur[1024];
    for (int i = threadIdx.x; i < HSLOTS; i += blockDim.x) keys[i] = -1;
    for (int k = threadIdx.x; k < jb; k += blockDim.x) {
        cur[k] = r0 + k;
        const long long rel = ipiv_rel[k];
        gpiv[k] = (rel >= k && r0 + rel < nrows ? rel : k) + goff;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 0; k < jb; ++k) {
            const long long rel = ipiv_rel[k];
            const long long p = rel >= k && r0 + rel < nrows ? r0 + rel : r0 + k;
            if (p == r0 + k) continue;
            if (p < r0 + jb) {
                const long long t = cur[k];
                cur[k] = cur[p - r0];
                cur[p - r0] = t;
            } else {
                unsigned h = (unsigned)((unsigned long long)p * 0x9E3779B97F4A7C15ull >> 53) &
                             (HSLOTS - 1);
                while (keys[h] != -1 && keys[h] != p) h = (h + 1) & (HSLOTS - 1);
                const long long content = keys[h] == p ? vals[h] : p;
                keys[h] = p;
                vals[h] = cur[k];
                cur[k] = content;
            }
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < jb; k += blockDim.x) src[k] = cur[k];
    // compact the displaced (dst, src) pairs in slot order (deterministic)
    if (threadIdx.x == 0) {
        int n = 0;
        for (int h = 0; h < HSLOTS; ++h)
            if (keys[h] != -1) {
                disp[2 * n] = keys[h];
                disp[2 * n + 1] = vals[h];
                ++n;
            }
        *ndisp = n;
    }
}

constexpr int LS_COLS = 64;      // columns per CTA (one warp covers 64 doubles with 16B lanes)
constexpr int LS_WARPS = 8;
constexpr int LS_UNROLL = 4;     // row copies in flight per warp (HBM latency x bandwidth)
constexpr int LS_MAXJB = 1024;

// One pass over columns [c0, c1) of the row swaps of one panel: every CTA
// first stages the plan (src rows, displaced pairs) in shared memory, then
// each warp moves LS_UNROLL rows at a time with 16-byte lanes (all loads of
// a group issued before its stores).  Phase 1 gathers the block's final
// rows into U; after a CTA barrier (every read of a displaced row precedes
// its overwrite) phase 2 writes the displaced rows.
__global__ void __launch_bounds__(LS_WARPS * 32)
laswp_gs_kernel(int jb, const int64_t *__restrict__ src, const int64_t *__restrict__ disp,
                const int *__restrict__ ndisp, double *A, long long lda, long long c0,
                long long c1, double *U, long long ldu, int vec)
{
    __shared__ long long s_src[LS_MAXJB];
    __shared__ long long s_dd[LS_MAXJB], s_ds[LS_MAXJB];
    const int nd = *ndisp;
    for (int k = threadIdx.x; k < jb; k += blockDim.x) s_src[k] = src[k];
    for (int d = threadIdx.x; d < nd; d += blockDim.x) {
        s_dd[d] = disp[2 * d];
        s_ds[d] = disp[2 * d + 1];
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long cb = c0 + (long long)blockIdx.x * LS_COLS;  // first column of this CTA
    const long long col = cb + 2 * lane;
    const bool has0 = col < c1, has1 = col + 1 < c1;
    auto move = [&](int total, auto srow, auto drow) {
        for (int k0 = warp * LS_UNROLL; k0 < total; k0 += LS_WARPS * LS_UNROLL) {
            if (vec && has1) {
                double2 v[LS_UNROLL];
#pragma unroll
                for (int u = 0; u < LS_UNROLL; ++u)
                    if (k0 + u < total)
                        v[u] = *reinterpret_cast<const double2 *>(srow(k0 + u));
#pragma unroll
                for (int u = 0; u < LS_UNROLL; ++u)
                    if (k0 + u < total) *reinterpret_cast<double2 *>(drow(k0 + u)) = v[u];
            } else {
                double v0[LS_UNROLL], v1[LS_UNROLL];
#pragma unroll
                for (int u = 0; u < LS_UNROLL; ++u)
                    if (k0 + u < total) {
                        v0[u] = has0 ? srow(k0 + u)[0] : 0.0;
                        v1[u] = has1 ? srow(k0 + u)[1] : 0.0;
                    }
#pragma unroll
                for (int u = 0; u < LS_UNROLL; ++u)
                    if (k0 + u < total) {
                        if (has0) drow(k0 + u)[0] = v0[u];
                        if (has1) drow(k0 + u)[1] = v1[u];
                    }
            }
        }
    };
    // (the accessors return this lane's element: A column col, U column col - c0)
    // phase 1: gather the block's final rows into U
    move(jb, [&](int k) -> const double * { return A + s_src[k] * lda + col; },
         [&](int k) -> double * { return U + (long long)k * ldu + (col - c0); });
    __syncthreads();
    // phase 2: displaced rows receive original block rows
    move(nd, [&](int d) -> const double * { return A + s_ds[d] * lda + col; },
         [&](int d) -> double * { return A + s_dd[d] * lda + col; });
}

// ---- P > 1: the row swaps cross process rows (RS over the column communicator)
__device__ __forceinline__ bool owns_row(long long g, int NB, int P, int myrow)
{
    return (int)((g / NB) % P) == myrow;
}
__device__ __forceinline__ long long g2l_row(long long g, int NB, int P)
{
    return (g / ((long long)NB * P)) * NB + g % NB;
}

// U[k][c] = A[local(src[k])][c0 + c] when this process row owns src[k], else 0
// (summed over the process column afterwards: every process gets all of U).
__global__ void __launch_bounds__(LS_WARPS * 32)
rs_pack_kernel(int jb, const int64_t *__restrict__ src, const double *__restrict__ A,
               long long lda, long long c0, long long c1, double *U, long long ldu, int NB, int P,
               int myrow)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long col = c0 + (long long)blockIdx.x * LS_COLS + 2 * lane;
    const bool has0 = col < c1, has1 = col + 1 < c1;
    for (int k = warp; k < jb; k += LS_WARPS) {
        const long long g = src[k];
        double *d = U + (long long)k * ldu + (col - c0);
        if (owns_row(g, NB, P, myrow)) {
            const double *sp = A + g2l_row(g, NB, P) * lda + col;
            if (has0) d[0] = sp[0];
            if (has1) d[1] = sp[1];
        } else {
            if (has0) d[0] = 0.0;
            if (has1) d[1] = 0.0;
        }
    }
}

// A[local(d)][c0 + c] = W[s - j0][c] for the displaced pairs (d, s) this process row owns;
// W holds the original block row j (from its owner).  The owned pairs are
// compacted in shared memory first, then LS_UNROLL rows per warp are in flight.
__global__ void __launch_bounds__(LS_WARPS * 32)
rs_scatter_kernel(const int64_t *__restrict__ disp, const int *__restrict__ ndisp,
                  const double *__restrict__ W, long long ldw, long long j0, double *A,
                  long long lda, long long c0, long long c1, int NB, int P, int myrow, int vec)
{
    __shared__ long long s_dst[LS_MAXJB], s_w[LS_MAXJB];   // s_dst < 0: not this process row's
    const int nd = *ndisp;
    for (int d = threadIdx.x; d < nd; d += blockDim.x) {
        const long long g = disp[2 * d];
        const bool mine = owns_row(g, NB, P, myrow);
        s_dst[d] = mine ? g2l_row(g, NB, P) : -1;
        s_w[d] = disp[2 * d + 1] - j0;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long col = c0 + (long long)blockIdx.x * LS_COLS + 2 * lane;
    const bool has0 = col < c1, has1 = col + 1 < c1;
    const int total = nd;
    for (int k0 = warp * LS_UNROLL; k0 < total; k0 += LS_WARPS * LS_UNROLL) {
        if (vec && has1) {
            double2 v[LS_UNROLL];
#pragma unroll
            for (int u = 0; u < LS_UNROLL; ++u)
                if (k0 + u < total && s_dst[k0 + u] >= 0)
                    v[u] = *reinterpret_cast<const double2 *>(W + s_w[k0 + u] * ldw + (col - c0));
#pragma unroll
            for (int u = 0; u < LS_UNROLL; ++u)
                if (k0 + u < total && s_dst[k0 + u] >= 0)
                    *reinterpret_cast<double2 *>(A + s_dst[k0 + u] * lda + col) = v[u];
        } else {
#pragma unroll
            for (int u = 0; u < LS_UNROLL; ++u)
                if (k0 + u < total && s_dst[k0 + u] >= 0) {
                    const double *sp = W + s_w[k0 + u] * ldw + (col - c0);
                    double *t = A + s_dst[k0 + u] * lda + col;
                    if (has0) t[0] = sp[0];
                    if (has1) t[1] = sp[1];
                }
        }
    }
}

// ---- P > 1 RS over peer memory (CUDA IPC over NVLink), no collective library.
// Every process of the column maps every peer's local A.  Phase 1 (after a
// flag barrier: every peer has finished updating these columns for
// iteration j): gather U[k] = row src[k] from its owner's A, and — for the
// displaced rows this process owns — the original block row they receive,
// from the owner of block row j, into W.  Phase 2 (after a second barrier:
// every peer has finished reading) is rs_scatter from W.
// lane p < P: announce arrival at `slot` to peer p, then wait (bounded) for
// peer p's arrival.
__global__ void rs_barrier_kernel(RsPeers pr, int slot, unsigned long long value, SpinCtl sc)
{
    const int p = threadIdx.x;
    if (p >= pr.P) return;
    __threadfence_system();
    st_release_sys(pr.flag[p] + (size_t)slot * MAX_P + pr.myrow, value);
    spin_geq_sys(pr.my_flag + (size_t)slot * MAX_P + p, value, sc,
                 SITE_RS_BARRIER | (unsigned long long)slot << 4 | (unsigned long long)p << 8);
    __threadfence_system();
}

// Generic flag step (LBCAST over peer memory): lanes < nsig publish sv to
// sig[lane] (after a system fence: this stream's earlier writes are visible
// first); lanes < nwait wait (bounded) until *wt[lane] >= wv.
__global__ void flag_kernel(FlagOp op, SpinCtl sc)
{
    const int l = threadIdx.x;
    if (l < op.nsig) {
        __threadfence_system();
        st_release_sys(op.sig[l], op.sv);
    }
    if (l < op.nwait) spin_geq_sys(op.wt[l], op.wv, sc, SITE_FLAG | (unsigned long long)l << 8);
    __threadfence_system();
}

// Phase 1 of the peer-memory RS: the plan (which row of which peer lands in
// which row of U or W) is resolved once per CTA into shared memory, then each
// warp keeps LS_UNROLL 16-byte row copies in flight (peer rows come over
// NVLink; the reads bypass L1: __ldcg).
__global__ void __launch_bounds__(LS_WARPS * 32)
rs_gather_peer_kernel(int jb, const int64_t *__restrict__ src, const int64_t *__restrict__ disp,
                      const int *__restrict__ ndisp, RsPeers pr, long long lda, long long c0,
                      long long c1, double *__restrict__ U, long long ldu,
                      double *__restrict__ W, long long ldw, long long j0, int NB, int vec)
{
    // entries [0, jb): U rows; [jb, jb + nd): displaced pairs (null when the
    // displaced row is not this process row's)
    __shared__ const double *s_src[2 * LS_MAXJB];
    __shared__ double *s_dst[2 * LS_MAXJB];
    const int P = pr.P;
    const int bowner = (int)((j0 / NB) % P);
    const int nd = *ndisp;
    for (int k = threadIdx.x; k < jb; k += blockDim.x) {
        const long long g = src[k];
        s_src[k] = pr.A[(int)((g / NB) % P)] + g2l_row(g, NB, P) * lda;
        s_dst[k] = U + (long long)k * ldu - c0;
    }
    for (int d = threadIdx.x; d < nd; d += blockDim.x) {
        const long long dg = disp[2 * d], sg = disp[2 * d + 1];
        const bool mine = owns_row(dg, NB, P, pr.myrow);
        s_src[jb + d] = mine ? pr.A[bowner] + g2l_row(sg, NB, P) * lda : nullptr;
        s_dst[jb + d] = W + (sg - j0) * ldw - c0;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long col = c0 + (long long)blockIdx.x * LS_COLS + 2 * lane;
    const bool has0 = col < c1, has1 = col + 1 < c1;
    const int total = jb + nd;
    for (int k0 = warp * LS_UNROLL; k0 < total; k0 += LS_WARPS * LS_UNROLL) {
        if (vec && has1) {
            double2 v[LS_UNROLL];
#pragma unroll
            for (int u = 0; u < LS_UNROLL; ++u)
                if (k0 + u < total && s_src[k0 + u])
                    v[u] = __ldcg(reinterpret_cast<const double2 *>(s_src[k0 + u] + col));
#pragma unroll
            for (int u = 0; u < LS_UNROLL; ++u)
                if (k0 + u < total && s_src[k0 + u])
                    *reinterpret_cast<double2 *>(s_dst[k0 + u] + col) = v[u];
        } else {
#pragma unroll
            for (int u = 0; u < LS_UNROLL; ++u)
                if (k0 + u < total && s_src[k0 + u]) {
                    const double *sp = s_src[k0 + u] + col;
                    double *dp = s_dst[k0 + u] + col;
                    if (has0) dp[0] = __ldcg(sp);
                    if (has1) dp[1] = __ldcg(sp + 1);
                }
        }
    }
}

}  // namespace

cudaError_t rs_pack(cudaStream_t st, int64_t jb, const int64_t *src, const double *A, int64_t lda,
                    int64_t c0, int64_t c1, double *U, int64_t ldu, int NB, int P, int myrow)
{
    if (jb <= 0 || c1 <= c0) return cudaSuccess;
    rs_pack_kernel<<<(unsigned)cdiv(c1 - c0, LS_COLS), LS_WARPS * 32, 0, st>>>(
        (int)jb, src, A, lda, c0, c1, U, ldu, NB, P, myrow);
    count_launch();
    return cudaGetLastError();
}

cudaError_t rs_scatter(cudaStream_t st, const int64_t *disp, const int *ndisp, const double *W,
                       int64_t ldw, int64_t j0, double *A, int64_t lda, int64_t c0, int64_t c1,
                       int NB, int P, int myrow)
{
    if (c1 <= c0) return cudaSuccess;
    const int vec = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(W)) & 15) == 0 &&
                    (lda & 1) == 0 && (ldw & 1) == 0 && (c0 & 1) == 0;
    rs_scatter_kernel<<<(unsigned)cdiv(c1 - c0, LS_COLS), LS_WARPS * 32, 0, st>>>(
        disp, ndisp, W, ldw, j0, A, lda, c0, c1, NB, P, myrow, vec);
    count_launch();
    return cudaGetLastError();
}

cudaError_t rs_barrier(cudaStream_t st, const RsPeers &pr, int slot, unsigned long long value,
                       const SpinCtl &sc)
{
    if (pr.P < 1 || pr.P > MAX_P || slot < 0 || slot >= RS_SLOTS) return cudaErrorInvalidValue;
    rs_barrier_kernel<<<1, 32, 0, st>>>(pr, slot, value, sc);
    count_launch();
    return cudaGetLastError();
}

cudaError_t rs_gather_peer(cudaStream_t st, int64_t jb, const int64_t *src, const int64_t *disp,
                           const int *ndisp, const RsPeers &pr, int64_t lda, int64_t c0,
                           int64_t c1, double *U, int64_t ldu, double *W, int64_t ldw, int64_t j0,
                           int NB)
{
    if (jb <= 0 || c1 <= c0) return cudaSuccess;
    if (jb > LS_MAXJB) return cudaErrorInvalidValue;
    bool vec = (lda & 1) == 0 && (c0 & 1) == 0 && (ldu & 1) == 0 && (ldw & 1) == 0 &&
               (reinterpret_cast<uintptr_t>(U) & 15) == 0 &&
               (reinterpret_cast<uintptr_t>(W) & 15) == 0;
    for (int p = 0; p < pr.P; ++p) vec = vec && (reinterpret_cast<uintptr_t>(pr.A[p]) & 15) == 0;
    rs_gather_peer_kernel<<<(unsigned)cdiv(c1 - c0, LS_COLS), LS_WARPS * 32, 0, st>>>(
        (int)jb, src, disp, ndisp, pr, lda, c0, c1, U, ldu, W, ldw, j0, NB, vec ? 1 : 0);
    count_launch();
    return cudaGetLastError();
}

cudaError_t flag_op(cudaStream_t st, const FlagOp &op, const SpinCtl &sc)
{
    if (op.nsig < 0 || op.nsig > 32 || op.nwait < 0 || op.nwait > 32) return cudaErrorInvalidValue;
    if (op.nsig == 0 && op.nwait == 0) return cudaSuccess;
    flag_kernel<<<1, 32, 0, st>>>(op, sc);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pivot_plan(cudaStream_t st, int64_t jb, int64_t r0, const int64_t *ipiv_rel,
                       int64_t goff, int64_t nrows, int64_t *gpiv, int64_t *src, int64_t *disp,
                       int *ndisp)
{
    if (jb <= 0) return cudaSuccess;
    if (jb > 1024) return cudaErrorInvalidValue;
    pivot_plan_kernel<<<1, 256, 0, st>>>((int)jb, r0, ipiv_rel, goff, nrows, gpiv, src, disp,
                                         ndisp);
    count_launch();
    return cudaGetLastError();
}

cudaError_t laswp_gather_scatter(cudaStream_t st, int64_t jb, const int64_t *src,
                                 const int64_t *disp, const int *ndisp, double *A, int64_t lda,
                                 int64_t c0, int64_t c1, double *U, int64_t ldu)
{
    if (jb <= 0 || c1 <= c0) return cudaSuccess;
    if (jb > LS_MAXJB) return cudaErrorInvalidValue;
    const int vec = ((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (lda & 1) == 0 &&
                     (c0 & 1) == 0 && (reinterpret_cast<uintptr_t>(U) & 15) == 0 &&
                     (ldu & 1) == 0)
                        ? 1
                        : 0;
    const int64_t nblk = cdiv(c1 - c0, LS_COLS);
    laswp_gs_kernel<<<(unsigned)nblk, LS_WARPS * 32, 0, st>>>((int)jb, src, disp, ndisp, A, lda,
                                                              c0, c1, U, ldu, vec);
    count_launch();
    return cudaGetLastError();
}

}  // namespace hpl
