// kernels_fact.cu — device panel FACT, no CPU fallback.
//
// The paper factors the tall-skinny M x NB panel on the CPU with T threads
// that own NB-row tiles round-robin, a parallel max-reduction for the pivot,
// the main thread applying the swap and all threads doing the rank-1 update
// of their own tiles, with the recursive right-looking
// variant, two subdivisions, base block 16 and a right-looking leaf
// (PAPER.md l.34).  Here the "threads" are CTAs of one cooperative kernel:
// each CTA owns a contiguous chunk of panel rows, finds its local pivot
// candidate with warp shuffles, publishes (|v|, row, the row's leaf values)
// — the payload travels with the reduction — and after ONE
// grid-wide barrier per column every CTA reduces the candidates itself,
// applies the swap to the rows it owns and updates them.  The recursion's
// TRSM and GEMM steps run as separate kernels (the GEMM is the DMMA kernel).
#include "hpl_internal.cuh"
#include <cooperative_groups.h>
#include <cstdio>
#include <mutex>

namespace hpl {

namespace {

constexpr int LEAF_MAX = 16;           // widest leaf (NBMIN)
constexpr int REC = 2 + LEAF_MAX;      // doubles per candidate record
constexpr int FACT_THREADS = 256;
constexpr int MAX_CTAS = 1024;

// Software grid barrier of the cooperative leaf (co-residency guaranteed by
// the cooperative launch).  Bounded like every other spin (SpinCtl): after
// an abort the CTAs leave it at once.
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned nblocks, const SpinCtl &sc)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g0 = *gen;
        __threadfence();
        const unsigned arrived = atomicAdd(bar, 1u);
        if (arrived == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            const unsigned long long t0 = gtimer();
            for (unsigned n = 1; *gen == g0; ++n) {
                if ((n & 63u) == 0) {
                    if (spin_aborted(sc)) break;
                    if (gtimer() - t0 > sc.timeout_ns) {
                        spin_record(sc, SITE_GRID_BARRIER, g0 + 1, *gen);
                        break;
                    }
                }
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// better(a, b): a beats b  <=>  |a| > |b|, ties -> smaller row (reading A2)
__device__ __forceinline__ bool better(double va, long long ra, double vb, long long rb)
{
    return va > vb || (va == vb && ra < rb);
}

__device__ __forceinline__ void warp_argmax(double &v, long long &r)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const long long orow = __shfl_xor_sync(0xffffffffu, r, o);
        if (better(ov, orow, v, r)) { v = ov; r = orow; }
    }
}

// Row update shared by both leaves: for panel row i, l = P[kc][i] / piv and
// P[k0+cc][i] -= l * prow[cc] for the leaf columns cc > kk.  All the row's
// loads are issued before any store (one L2 round trip instead of one per
// column); returns the new |P[kc+1][i]| for the next column's pivot search.
__device__ __forceinline__ double leaf_row_update(double *P, int64_t ldp, int k0, int w, int kk,
                                                  int64_t i, double piv, const double *prow)
{
    const int kc = k0 + kk;
    const double xk = P[(int64_t)kc * ldp + i];
    double v[LEAF_MAX];
#pragma unroll
    for (int c = 0; c < LEAF_MAX; ++c) {
        const int cc = kk + 1 + c;
        v[c] = cc < w ? P[(int64_t)(k0 + cc) * ldp + i] : 0.0;
    }
    const double l = xk / piv;
    P[(int64_t)kc * ldp + i] = l;
#pragma unroll
    for (int c = 0; c < LEAF_MAX; ++c) {
        const int cc = kk + 1 + c;
        if (cc < w) {
            v[c] = fma(-l, prow[cc], v[c]);
            P[(int64_t)(k0 + cc) * ldp + i] = v[c];
        }
    }
    return fabs(v[0]);
}

// Two rows (i0 and i1 = i0 + stride) at once: both rows' loads are issued
// before either row's stores, twice the loads in flight per thread (a leaf
// on few CTAs is bound by each SM's outstanding loads).  The arithmetic per
// row is leaf_row_update's, so the bits are the same.
__device__ __forceinline__ void leaf_row_update2(double *P, int64_t ldp, int k0, int w, int kk,
                                                 int64_t i0, int64_t i1, double piv,
                                                 const double *prow, double &n0, double &n1)
{
    const int kc = k0 + kk;
    const double x0 = P[(int64_t)kc * ldp + i0], x1 = P[(int64_t)kc * ldp + i1];
    double v0[LEAF_MAX], v1[LEAF_MAX];
#pragma unroll
    for (int c = 0; c < LEAF_MAX; ++c) {
        const int cc = kk + 1 + c;
        v0[c] = cc < w ? P[(int64_t)(k0 + cc) * ldp + i0] : 0.0;
        v1[c] = cc < w ? P[(int64_t)(k0 + cc) * ldp + i1] : 0.0;
    }
    const double l0 = x0 / piv, l1 = x1 / piv;
    P[(int64_t)kc * ldp + i0] = l0;
    P[(int64_t)kc * ldp + i1] = l1;
#pragma unroll
    for (int c = 0; c < LEAF_MAX; ++c) {
        const int cc = kk + 1 + c;
        if (cc < w) {
            v0[c] = fma(-l0, prow[cc], v0[c]);
            v1[c] = fma(-l1, prow[cc], v1[c]);
            P[(int64_t)(k0 + cc) * ldp + i0] = v0[c];
            P[(int64_t)(k0 + cc) * ldp + i1] = v1[c];
        }
    }
    n0 = fabs(v0[0]);
    n1 = fabs(v1[0]);
}

// Leaf: right-looking GEPP of columns [k0, k0+w) of the panel (rows k0..m-1).
// One grid barrier per column; the next column's local pivot candidate is
// formed during the current column's update, so a column costs the barrier
// plus about three L2 round trips.
// NT = 256: the leaf on its own SMs (FACT on the critical path).  NT = 32:
// one warp per CTA, at most 128 registers, so a leaf CTA fits on an SM next
// to three trailing-DGEMM CTAs (3 x 160 threads x 128 registers + 32 x 128 =
// the 64 K register file) and takes no DGEMM slot while FACT hides behind it.
template <int NT>
__global__ void __launch_bounds__(NT, NT == 32 ? 16 : 1)
leaf_fact_kernel(int m, int64_t ldp, double *P, int k0, int w, int64_t *ipiv, double *cand,
                 unsigned *bar, unsigned long long *info, long long goff, SpinCtl sc)
{
    const unsigned G = gridDim.x;
    const int nrows = m - k0;
    const int chunk = (nrows + (int)G - 1) / (int)G;
    const int rbeg = k0 + (int)blockIdx.x * chunk;
    const int rend = min(m, rbeg + chunk);
    __shared__ double s_v[NT / 32];
    __shared__ long long s_r[NT / 32];
    __shared__ int s_c[NT / 32];
    __shared__ double s_prow[LEAF_MAX], s_rowk[LEAF_MAX];
    __shared__ long long s_p;
    __shared__ double s_piv;

    // local candidate for the first leaf column
    double bv = -1.0;
    long long br = LLONG_MAX;
    for (int i = max(rbeg, k0) + threadIdx.x; i < rend; i += NT) {
        const double v = fabs(P[(int64_t)k0 * ldp + i]);
        if (better(v, i, bv, br)) { bv = v; br = i; }
    }
    for (int kk = 0; kk < w; ++kk) {
        const int kc = k0 + kk;
        double *rec = cand + (size_t)(kk & 1) * (MAX_CTAS + 1) * REC;
        // ---- 1. this CTA's candidate: (|v|, row, the row's leaf values)
        warp_argmax(bv, br);
        if ((threadIdx.x & 31) == 0) { s_v[threadIdx.x >> 5] = bv; s_r[threadIdx.x >> 5] = br; }
        __syncthreads();
        if (threadIdx.x < 32) {
            bv = threadIdx.x < NT / 32 ? s_v[threadIdx.x] : -1.0;
            br = threadIdx.x < NT / 32 ? s_r[threadIdx.x] : LLONG_MAX;
            warp_argmax(bv, br);
            double *myrec = rec + (size_t)blockIdx.x * REC;
            if (threadIdx.x == 0) {
                myrec[0] = bv;
                myrec[1] = __longlong_as_double(br);
            }
            if (br != LLONG_MAX && threadIdx.x < w)
                myrec[2 + threadIdx.x] = P[(int64_t)(k0 + threadIdx.x) * ldp + br];
            if (kc >= rbeg && kc < rend && threadIdx.x < w)
                rec[(size_t)G * REC + 2 + threadIdx.x] = P[(int64_t)(k0 + threadIdx.x) * ldp + kc];
        }
        __threadfence();
        grid_barrier(bar, G, sc);

        // ---- 2. every CTA reduces all candidates (deterministic)
        bv = -1.0;
        br = LLONG_MAX;
        int bc = -1;
        for (int c = threadIdx.x; c < (int)G; c += NT) {
            // other CTAs wrote these: read through L2 (L1 is not coherent)
            const double v = __ldcg(rec + (size_t)c * REC);
            const long long r = __double_as_longlong(__ldcg(rec + (size_t)c * REC + 1));
            if (r != LLONG_MAX && better(v, r, bv, br)) { bv = v; br = r; bc = c; }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const long long orow = __shfl_xor_sync(0xffffffffu, br, o);
            const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
            if (better(ov, orow, bv, br)) { bv = ov; br = orow; bc = oc; }
        }
        if ((threadIdx.x & 31) == 0) {
            s_v[threadIdx.x >> 5] = bv; s_r[threadIdx.x >> 5] = br; s_c[threadIdx.x >> 5] = bc;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const bool ok = threadIdx.x < NT / 32;
            bv = ok ? s_v[threadIdx.x] : -1.0;
            br = ok ? s_r[threadIdx.x] : LLONG_MAX;
            bc = ok ? s_c[threadIdx.x] : -1;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const long long orow = __shfl_xor_sync(0xffffffffu, br, o);
                const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
                if (better(ov, orow, bv, br)) { bv = ov; br = orow; bc = oc; }
            }
            // (bc < 0 only if no CTA reported a candidate: after an abandoned
            // barrier; read a valid slot, the pivot is discarded downstream)
            if (bc < 0) bc = 0;
            if (threadIdx.x == 0) {
                s_p = br;
                s_piv = __ldcg(rec + (size_t)bc * REC + 2 + kk);
            }
            if (threadIdx.x < w) {
                s_prow[threadIdx.x] = __ldcg(rec + (size_t)bc * REC + 2 + threadIdx.x);
                s_rowk[threadIdx.x] = __ldcg(rec + (size_t)G * REC + 2 + threadIdx.x);
            }
        }
        __syncthreads();
        const long long p = s_p;
        const double piv = s_piv;
        if (threadIdx.x == 0 && blockIdx.x == 0) {
            ipiv[kc] = p;
            if (piv == 0.0) atomicMin(info, (unsigned long long)(goff + kc));
        }
        // ---- 3. swap rows kc and p inside the leaf columns (owners only)
        if (p != kc) {
            if (kc >= rbeg && kc < rend && threadIdx.x < w)
                P[(int64_t)(k0 + threadIdx.x) * ldp + kc] = s_prow[threadIdx.x];
            if (p >= rbeg && p < rend && threadIdx.x < w)
                P[(int64_t)(k0 + threadIdx.x) * ldp + p] = s_rowk[threadIdx.x];
        }
        __syncthreads();
        // ---- 4. scale + rank-1 update of own rows > kc; next column's candidate
        bv = -1.0;
        br = LLONG_MAX;
        int i = max(rbeg, kc + 1) + threadIdx.x;
        if (NT > 32) {
            for (; i + NT < rend; i += 2 * NT) {
                double n0, n1;
                leaf_row_update2(P, ldp, k0, w, kk, i, i + NT, piv, s_prow, n0, n1);
                if (kk + 1 < w && better(n0, i, bv, br)) { bv = n0; br = i; }
                if (kk + 1 < w && better(n1, i + NT, bv, br)) { bv = n1; br = i + NT; }
            }
        }
        for (; i < rend; i += NT) {
            const double nv = leaf_row_update(P, ldp, k0, w, kk, i, piv, s_prow);
            if (kk + 1 < w && better(nv, i, bv, br)) { bv = nv; br = i; }
        }
    }
}

// Left-looking and Crout leaves (rocHPL's FACT variants;
// SURVEY §8(f) NEXT 3).  Same grid, same one barrier per column and the same
// pivot rule as leaf_fact_kernel; only the data flow differs:
//  - the column kk is brought up to date only when it is reached:
//    v_i = a_i,kk - sum_{c<kk} l_i,c u_c,kk (FMAs in ascending c), fused with
//    the scaling of column kk-1 for the CTA's own rows;
//  - the U rows of the leaf are formed in shared memory by every CTA from the
//    broadcast pivot rows: u_kk,cc = p_cc - sum_{c<kk} p_c u_c,cc;
//  - LEFT writes u_c,kk into the rows above when column kk is reached
//    (column-by-column triangular solve), CROUT writes the whole U row kk at
//    its pivot step.
// Each result goes through the same FMA sequence with the same operands as
// the right-looking leaf's in-place updates, so all three are bitwise equal
// (tested), and differ only in memory traffic and timing.
template <int NT, bool CROUT>
__global__ void __launch_bounds__(NT, 1)
leaf_fact_ll_kernel(int m, int64_t ldp, double *P, int k0, int w, int64_t *ipiv, double *cand,
                    unsigned *bar, unsigned long long *info, long long goff, SpinCtl sc)
{
    const unsigned G = gridDim.x;
    const int nrows = m - k0;
    const int chunk = (nrows + (int)G - 1) / (int)G;
    const int rbeg = k0 + (int)blockIdx.x * chunk;
    const int rend = min(m, rbeg + chunk);
    __shared__ double s_v[NT / 32];
    __shared__ long long s_r[NT / 32];
    __shared__ int s_c[NT / 32];
    __shared__ double s_prow[LEAF_MAX], s_rowk[LEAF_MAX];
    __shared__ double s_U[LEAF_MAX][LEAF_MAX];
    __shared__ long long s_p;
    __shared__ double s_piv;

    double bv = -1.0;
    long long br = LLONG_MAX;
    for (int i = max(rbeg, k0) + threadIdx.x; i < rend; i += NT) {
        const double v = fabs(P[(int64_t)k0 * ldp + i]);
        if (better(v, i, bv, br)) { bv = v; br = i; }
    }
    for (int kk = 0; kk < w; ++kk) {
        const int kc = k0 + kk;
        double *rec = cand + (size_t)(kk & 1) * (MAX_CTAS + 1) * REC;
        // ---- LEFT: the rows above reach column kk (u_c,kk, c < kk, from s_U)
        if (!CROUT)
            for (int c = threadIdx.x; c < kk; c += NT)
                if (k0 + c >= rbeg && k0 + c < rend)
                    P[(int64_t)kc * ldp + k0 + c] = s_U[c][kk];
        // ---- 1. candidate record (|v|, row, the row's current leaf values)
        warp_argmax(bv, br);
        if ((threadIdx.x & 31) == 0) { s_v[threadIdx.x >> 5] = bv; s_r[threadIdx.x >> 5] = br; }
        __syncthreads();
        if (threadIdx.x < 32) {
            bv = threadIdx.x < NT / 32 ? s_v[threadIdx.x] : -1.0;
            br = threadIdx.x < NT / 32 ? s_r[threadIdx.x] : LLONG_MAX;
            warp_argmax(bv, br);
            double *myrec = rec + (size_t)blockIdx.x * REC;
            if (threadIdx.x == 0) {
                myrec[0] = bv;
                myrec[1] = __longlong_as_double(br);
            }
            if (br != LLONG_MAX && threadIdx.x < w)
                myrec[2 + threadIdx.x] = P[(int64_t)(k0 + threadIdx.x) * ldp + br];
            if (kc >= rbeg && kc < rend && threadIdx.x < w)
                rec[(size_t)G * REC + 2 + threadIdx.x] = P[(int64_t)(k0 + threadIdx.x) * ldp + kc];
        }
        __threadfence();
        grid_barrier(bar, G, sc);

        // ---- 2. every CTA reduces all candidates (deterministic)
        bv = -1.0;
        br = LLONG_MAX;
        int bc = -1;
        for (int c = threadIdx.x; c < (int)G; c += NT) {
            const double v = __ldcg(rec + (size_t)c * REC);
            const long long r = __double_as_longlong(__ldcg(rec + (size_t)c * REC + 1));
            if (r != LLONG_MAX && better(v, r, bv, br)) { bv = v; br = r; bc = c; }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const long long orow = __shfl_xor_sync(0xffffffffu, br, o);
            const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
            if (better(ov, orow, bv, br)) { bv = ov; br = orow; bc = oc; }
        }
        if ((threadIdx.x & 31) == 0) {
            s_v[threadIdx.x >> 5] = bv; s_r[threadIdx.x >> 5] = br; s_c[threadIdx.x >> 5] = bc;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const bool ok = threadIdx.x < NT / 32;
            bv = ok ? s_v[threadIdx.x] : -1.0;
            br = ok ? s_r[threadIdx.x] : LLONG_MAX;
            bc = ok ? s_c[threadIdx.x] : -1;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const long long orow = __shfl_xor_sync(0xffffffffu, br, o);
                const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
                if (better(ov, orow, bv, br)) { bv = ov; br = orow; bc = oc; }
            }
            // (bc < 0 only if no CTA reported a candidate: after an abandoned
            // barrier; read a valid slot, the pivot is discarded downstream)
            if (bc < 0) bc = 0;
            if (threadIdx.x == 0) {
                s_p = br;
                s_piv = __ldcg(rec + (size_t)bc * REC + 2 + kk);
            }
            if (threadIdx.x < w) {
                s_prow[threadIdx.x] = __ldcg(rec + (size_t)bc * REC + 2 + threadIdx.x);
                s_rowk[threadIdx.x] = __ldcg(rec + (size_t)G * REC + 2 + threadIdx.x);
            }
        }
        __syncthreads();
        // ---- 3. U row kk: u_kk,cc = p_cc - sum_{c<kk} l_p,c u_c,cc (every CTA)
        if (threadIdx.x < w) {
            const int cc = threadIdx.x;
            double u = s_prow[cc];
            if (cc > kk)
                for (int c = 0; c < kk; ++c) u = fma(-s_prow[c], s_U[c][cc], u);
            s_U[kk][cc] = u;
        }
        __syncthreads();
        const long long p = s_p;
        const double piv = s_piv;
        if (threadIdx.x == 0 && blockIdx.x == 0) {
            ipiv[kc] = p;
            if (piv == 0.0) atomicMin(info, (unsigned long long)(goff + kc));
        }
        // ---- 4. swap rows kc and p inside the leaf columns (owners); CROUT
        // stores the finished U row kk into row kc right away
        if (kc >= rbeg && kc < rend && threadIdx.x < w)
            P[(int64_t)(k0 + threadIdx.x) * ldp + kc] =
                (CROUT && threadIdx.x > kk) ? s_U[kk][threadIdx.x] : s_prow[threadIdx.x];
        if (p != kc && p >= rbeg && p < rend && threadIdx.x < w)
            P[(int64_t)(k0 + threadIdx.x) * ldp + p] = s_rowk[threadIdx.x];
        __syncthreads();
        // ---- 5. own rows > kc: scale column kk; bring column kk+1 up to date
        // (one load per needed column, all before the stores); next candidate
        bv = -1.0;
        br = LLONG_MAX;
        const bool more = kk + 1 < w;
        for (int i = max(rbeg, kc + 1) + threadIdx.x; i < rend; i += NT) {
            double x[LEAF_MAX];
#pragma unroll
            for (int c = 0; c < LEAF_MAX; ++c)
                x[c] = (c <= kk + 1 && c < w) ? P[(int64_t)(k0 + c) * ldp + i] : 0.0;
            double l = 0.0;
#pragma unroll
            for (int c = 0; c < LEAF_MAX; ++c)
                if (c == kk) l = x[c] / piv;
            P[(int64_t)kc * ldp + i] = l;
            if (more) {
                double v = 0.0;
#pragma unroll
                for (int c = 0; c < LEAF_MAX; ++c)
                    if (c == kk + 1) v = x[c];
#pragma unroll
                for (int c = 0; c < LEAF_MAX; ++c)
                    if (c <= kk) v = fma(-(c == kk ? l : x[c]), s_U[c][kk + 1], v);
                P[(int64_t)(kc + 1) * ldp + i] = v;
                if (better(fabs(v), i, bv, br)) { bv = fabs(v); br = i; }
            }
        }
    }
    // LEFT: nothing is pending (column w-1's U entries were written at step w-1)
}

// Apply the leaf's swaps (ipiv[k0..k0+w), panel-relative) to the panel columns
// outside the leaf, dlaswp semantics.  Thread 0 turns the <= 16 sequential
// swaps into "row r receives the old content of row s" moves (as pivot_plan
// does for the trailing matrix); each thread then moves its column's rows
// with all loads issued before the stores.
__global__ void panel_laswp_kernel(int m, int nb, int64_t ldp, double *P, int k0, int w,
                                   const int64_t *ipiv)
{
    __shared__ long long s_dst[2 * LEAF_MAX], s_src[2 * LEAF_MAX];
    __shared__ int s_n;
    if (threadIdx.x == 0) {
        long long topc[LEAF_MAX], lowr[LEAF_MAX], lowc[LEAF_MAX];
        int nlow = 0;
        for (int t = 0; t < w; ++t) topc[t] = k0 + t;
        for (int t = 0; t < w; ++t) {
            const long long pp = ipiv[k0 + t];
            // (a pivot outside [k0+t, m) only follows an aborted leaf: skipped)
            if (pp == k0 + t || pp < k0 + t || pp >= m) continue;
            if (pp < k0 + w) {
                const long long tmp = topc[t];
                topc[t] = topc[pp - k0];
                topc[pp - k0] = tmp;
            } else {
                int f = -1;
                for (int q = 0; q < nlow; ++q)
                    if (lowr[q] == pp) f = q;
                const long long content = f >= 0 ? lowc[f] : pp;
                if (f >= 0) lowc[f] = topc[t];
                else { lowr[nlow] = pp; lowc[nlow] = topc[t]; ++nlow; }
                topc[t] = content;
            }
        }
        int n = 0;
        for (int t = 0; t < w; ++t)
            if (topc[t] != k0 + t) { s_dst[n] = k0 + t; s_src[n] = topc[t]; ++n; }
        for (int q = 0; q < nlow; ++q) { s_dst[n] = lowr[q]; s_src[n] = lowc[q]; ++n; }
        s_n = n;
    }
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nb || (c >= k0 && c < k0 + w)) return;
    double *col = P + (int64_t)c * ldp;
    const int n = s_n;
    double v[2 * LEAF_MAX];
#pragma unroll
    for (int q = 0; q < 2 * LEAF_MAX; ++q)
        if (q < n) v[q] = col[s_src[q]];
#pragma unroll
    for (int q = 0; q < 2 * LEAF_MAX; ++q)
        if (q < n) col[s_dst[q]] = v[q];
}

// ---------------------------------------------------------------- P > 1 leaf
// Leaf of the distributed panel: as leaf_fact_kernel, but the candidate search
// spans the process column.  Per column: local candidates -> grid barrier ->
// CTA 0 publishes (|v|, global row, the full panel row) into every peer's
// record slot and raises its flag, waits for all P flags, picks the winner
// (max |v|, smallest global row) and snapshots the replicated top row kc ->
// grid barrier -> full-width swap on the owners -> rank-1 update of the leaf
// columns.  The top block T is replicated on all P processes and updated
// identically by each, so only the winner's payload crosses NVLink.
template <int NT>
__global__ void __launch_bounds__(NT, NT == 32 ? 16 : 1)
leaf_fact_dist_kernel(int m, int64_t ldp, double *Pn, int k0, int w, int64_t *ipiv, double *cand,
                      double *win, double *tsnap, unsigned long long *winflag, unsigned *bar,
                      unsigned long long *info, DistPanel dp, DistExchange ex,
                      unsigned long long seq0, SpinCtl sc)
{
    const unsigned G = gridDim.x;
    const int chunk = (m + (int)G - 1) / (int)G;
    const int rbeg = (int)blockIdx.x * chunk;
    const int rend = min(m, rbeg + chunk);
    const int jbp = dp.jbp;
    __shared__ double s_v[NT / 32];
    __shared__ long long s_g[NT / 32];
    __shared__ int s_r[NT / 32];
    __shared__ double s_pay[1024], s_ts[1024];
    __shared__ long long s_win;
    auto grow = [&](int r) -> long long {
        if (r < jbp) return dp.j0 + r;
        const long long l = dp.lrL0 + (r - jbp);
        return ((l / dp.NB) * dp.P + dp.myrow) * dp.NB + l % dp.NB;
    };
    // Panel rows are ordered like their global rows (T = block row j first,
    // then this process's rows below it in block-cyclic order, a monotone
    // map), so ties are broken on the panel row and the global row is formed
    // once per CTA instead of per element.  T rows are candidates on the
    // owner of block row j only.
    double bv = -1.0;
    long long br = LLONG_MAX;
    for (int r = max(rbeg, k0) + threadIdx.x; r < rend; r += NT) {
        if (r < jbp && !dp.is_prow) continue;
        const double v = fabs(Pn[(int64_t)k0 * ldp + r]);
        if (better(v, r, bv, br)) { bv = v; br = r; }
    }
    for (int kk = 0; kk < w; ++kk) {
        const int kc = k0 + kk;
        const unsigned long long seq = seq0 + kk + 1;
        const int par = (int)(seq & 1);
        double *rec = cand + (size_t)(kk & 1) * (MAX_CTAS + 1) * REC;
        // ---- 1. this CTA's candidate (formed during the previous column's update)
        long long bg;
        warp_argmax(bv, br);
        if ((threadIdx.x & 31) == 0) { s_v[threadIdx.x >> 5] = bv; s_g[threadIdx.x >> 5] = br; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 1; q < NT / 32; ++q)
                if (better(s_v[q], s_g[q], bv, br)) { bv = s_v[q]; br = s_g[q]; }
            bg = br != LLONG_MAX ? grow((int)br) : LLONG_MAX;
            double *myrec = rec + (size_t)blockIdx.x * REC;
            myrec[0] = bv;
            myrec[1] = __longlong_as_double(bg);
            myrec[2] = __longlong_as_double(br != LLONG_MAX ? br : -1ll);
        }
        int brr;
        __threadfence();
        grid_barrier(bar, G, sc);

        // ---- 3. CTA 0: process-column exchange.  The other CTAs wait on the
        // local "winner ready" flag instead of a second grid barrier.
        if (blockIdx.x == 0) {
            if (threadIdx.x < 32) {
                bv = -1.0; bg = LLONG_MAX; brr = -1;
                for (unsigned c = threadIdx.x; c < G; c += 32) {
                    const double v = __ldcg(rec + (size_t)c * REC);
                    const long long g = __double_as_longlong(__ldcg(rec + (size_t)c * REC + 1));
                    const int r = (int)__double_as_longlong(__ldcg(rec + (size_t)c * REC + 2));
                    if (g != LLONG_MAX && better(v, g, bv, bg)) { bv = v; bg = g; brr = r; }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                    const long long og = __shfl_xor_sync(0xffffffffu, bg, o);
                    const int orr = __shfl_xor_sync(0xffffffffu, brr, o);
                    if (better(ov, og, bv, bg)) { bv = ov; bg = og; brr = orr; }
                }
                if (threadIdx.x == 0) { s_v[0] = bv; s_g[0] = bg; s_r[0] = brr; }
            }
            __syncthreads();
            bv = s_v[0]; bg = s_g[0]; brr = s_r[0];
            const size_t slot = ((size_t)par * ex.P + ex.myrow) * ex.recd;
            for (int c = threadIdx.x; c < jbp; c += NT) {
                const double pv = brr >= 0 ? __ldcg(Pn + (int64_t)c * ldp + brr) : 0.0;
                for (int p = 0; p < ex.P; ++p) ex.rec[p][slot + 2 + c] = pv;
                tsnap[c] = __ldcg(Pn + (int64_t)c * ldp + kc);
            }
            if (threadIdx.x == 0)
                for (int p = 0; p < ex.P; ++p) {
                    ex.rec[p][slot] = bv;
                    ex.rec[p][slot + 1] = __longlong_as_double(bg);
                }
            // bar.sync orders every thread's payload stores before the
            // system-scope release of the flag (cumulativity)
            __syncthreads();
            if (threadIdx.x < ex.P) {
                // flags of one parity slot only grow (seq advances by 2 between
                // its uses) and no peer can pass column seq before this one
                // published it, so ">= seq" is "== seq"
                st_release_sys(ex.flag[threadIdx.x] + (size_t)par * ex.P + ex.myrow, seq);
                spin_geq_sys(ex.my_flag + (size_t)par * ex.P + threadIdx.x, seq, sc,
                             SITE_DIST_PEER | (unsigned long long)threadIdx.x << 8);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int wslot = -1;
                bv = -1.0; bg = LLONG_MAX;
                for (int p = 0; p < ex.P; ++p) {
                    const double *r = ex.my_rec + ((size_t)par * ex.P + p) * ex.recd;
                    const double v = __ldcv(r);
                    const long long g = __double_as_longlong(__ldcv(r + 1));
                    if (g != LLONG_MAX && better(v, g, bv, bg)) { bv = v; bg = g; wslot = p; }
                }
                s_r[0] = wslot < 0 ? ex.myrow : wslot;   // (< 0 only after an abort)
                s_win = bg;
                win[0] = __longlong_as_double(bg);
            }
            __syncthreads();
            const double *wr = ex.my_rec + ((size_t)par * ex.P + s_r[0]) * ex.recd;
            for (int c = threadIdx.x; c < jbp; c += NT) {
                const double v = __ldcv(wr + 2 + c);
                win[2 + c] = v;
                s_pay[c] = v;
                s_ts[c] = tsnap[c];
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                st_release_gpu(winflag, seq);
            }
        } else {
            if (threadIdx.x == 0) spin_geq_gpu(winflag, seq, sc, SITE_DIST_WIN);
            __syncthreads();
            if (threadIdx.x == 0) s_win = __double_as_longlong(__ldcg(win));
            for (int c = threadIdx.x; c < jbp; c += NT) {
                s_pay[c] = __ldcg(win + 2 + c);
                s_ts[c] = __ldcg(tsnap + c);
            }
        }
        __syncthreads();

        // ---- 5. full-width swap on the owners of the two rows
        const long long gw = s_win;
        const long long t = gw - dp.j0;
        if (kc >= rbeg && kc < rend)
            for (int c = threadIdx.x; c < jbp; c += NT) Pn[(int64_t)c * ldp + kc] = s_pay[c];
        long long rswap = -1;
        if (t >= 0 && t < jbp) {
            if (t != kc) rswap = t;
        } else if ((int)((gw / dp.NB) % dp.P) == dp.myrow) {
            const long long l = (gw / ((long long)dp.NB * dp.P)) * dp.NB + gw % dp.NB;
            rswap = jbp + (l - dp.lrL0);
        }
        if (rswap >= rbeg && rswap < rend)
            for (int c = threadIdx.x; c < jbp; c += NT) Pn[(int64_t)c * ldp + rswap] = s_ts[c];
        const double piv = s_pay[kc];
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ipiv[kc] = t;
            if (piv == 0.0) atomicMin(info, (unsigned long long)(dp.j0 + kc));
        }
        __syncthreads();
        // ---- 6. scale column kc and rank-1 update of the leaf columns (own
        // rows > kc); the next column's local candidate on the way
        bv = -1.0;
        br = LLONG_MAX;
        const bool more = kk + 1 < w;
        int r = max(rbeg, kc + 1) + threadIdx.x;
        if (NT > 32) {
            for (; r + NT < rend; r += 2 * NT) {
                double n0, n1;
                leaf_row_update2(Pn, ldp, k0, w, kk, r, r + NT, piv, s_pay + k0, n0, n1);
                if (more && (r >= jbp || dp.is_prow) && better(n0, r, bv, br)) { bv = n0; br = r; }
                if (more && (r + NT >= jbp || dp.is_prow) && better(n1, r + NT, bv, br)) {
                    bv = n1;
                    br = r + NT;
                }
            }
        }
        for (; r < rend; r += NT) {
            const double nv = leaf_row_update(Pn, ldp, k0, w, kk, r, piv, s_pay + k0);
            if (more && (r >= jbp || dp.is_prow) && better(nv, r, bv, br)) { bv = nv; br = r; }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- cluster leaf (small panels)
// For panels of at most CL_SIZE x CL_ROWS rows (the tail, where FACT is on the
// critical path): ONE thread-block cluster factors the leaf with its w
// columns resident in shared memory (CL_ROWS rows per CTA), the candidate
// records written into every CTA's shared memory through DSMEM and one
// hardware cluster barrier per column — no L2 round trips per column, no
// grid-wide software barrier.  Same candidate rule and the same per-row
// operations as leaf_fact_kernel (bitwise-equal results, tested).
namespace cg = cooperative_groups;
constexpr int CL_SIZE = 16;           // non-portable cluster size (B200 allows 16)
constexpr int CL_THREADS = 512;
constexpr int CL_ROWS = 1664;         // rows per CTA: 1664 x 16 x 8 B = 208 KB of slab

__global__ void __launch_bounds__(CL_THREADS, 1)
leaf_fact_cluster_kernel(int m, int64_t ldp, double *P, int k0, int w, int64_t *ipiv,
                         unsigned long long *info, long long goff, int chunk)
{
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int CS = (int)cl.num_blocks();
    extern __shared__ double slab[];                 // slab[c * chunk + r]
    __shared__ double recs[2][CL_SIZE][REC];         // (|v|, row, row's leaf values) per CTA
    __shared__ double rowk[2][LEAF_MAX];             // row kc's leaf values (from its owner)
    __shared__ double s_v[CL_THREADS / 32];
    __shared__ long long s_r[CL_THREADS / 32];
    __shared__ double s_prow[LEAF_MAX], s_rowk[LEAF_MAX];
    __shared__ long long s_p;
    __shared__ double s_piv;
    const int tid = threadIdx.x;
    const int rbeg = k0 + rank * chunk;
    const int rend = min(m, rbeg + chunk);
    const int nr = max(0, rend - rbeg);
    for (int c = 0; c < w; ++c)
        for (int r = tid; r < nr; r += CL_THREADS)
            slab[c * chunk + r] = P[(int64_t)(k0 + c) * ldp + rbeg + r];
    __syncthreads();
    double bv = -1.0;
    long long br = LLONG_MAX;
    for (int r = tid; r < nr; r += CL_THREADS) {
        const double v = fabs(slab[r]);
        if (better(v, rbeg + r, bv, br)) { bv = v; br = rbeg + r; }
    }
    for (int kk = 0; kk < w; ++kk) {
        const int kc = k0 + kk, par = kk & 1;
        // ---- 1. this CTA's candidate, written into every CTA of the cluster
        warp_argmax(bv, br);
        if ((tid & 31) == 0) { s_v[tid >> 5] = bv; s_r[tid >> 5] = br; }
        __syncthreads();
        if (tid < 32) {
            bv = tid < CL_THREADS / 32 ? s_v[tid] : -1.0;
            br = tid < CL_THREADS / 32 ? s_r[tid] : LLONG_MAX;
            warp_argmax(bv, br);
            // lanes write the record's words to every destination CTA
            for (int e = tid; e < CS * (2 + LEAF_MAX); e += 32) {
                const int dst = e / (2 + LEAF_MAX), q = e % (2 + LEAF_MAX);
                double val;
                if (q == 0) val = bv;
                else if (q == 1) val = __longlong_as_double(br);
                else val = (br != LLONG_MAX && q - 2 < w) ? slab[(q - 2) * chunk + (br - rbeg)] : 0.0;
                double *d = cl.map_shared_rank(&recs[par][rank][q], dst);
                *d = val;
            }
            if (kc >= rbeg && kc < rend)
                for (int e = tid; e < CS * LEAF_MAX; e += 32) {
                    const int dst = e / LEAF_MAX, q = e % LEAF_MAX;
                    double *d = cl.map_shared_rank(&rowk[par][q], dst);
                    *d = q < w ? slab[q * chunk + (kc - rbeg)] : 0.0;
                }
        }
        cl.sync();
        // ---- 2. every CTA reduces the CS records (same order: same winner)
        if (tid < 32) {
            bv = -1.0;
            br = LLONG_MAX;
            int bc = -1;
            if (tid < CS) {
                const double v = recs[par][tid][0];
                const long long r = __double_as_longlong(recs[par][tid][1]);
                if (r != LLONG_MAX) { bv = v; br = r; bc = tid; }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const long long orow = __shfl_xor_sync(0xffffffffu, br, o);
                const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
                if (better(ov, orow, bv, br)) { bv = ov; br = orow; bc = oc; }
            }
            if (tid == 0) { s_p = br; s_piv = recs[par][bc][2 + kk]; }
            if (tid < w) {
                s_prow[tid] = recs[par][bc][2 + tid];
                s_rowk[tid] = rowk[par][tid];
            }
        }
        __syncthreads();
        const long long p = s_p;
        const double piv = s_piv;
        if (tid == 0 && rank == 0) {
            ipiv[kc] = p;
            if (piv == 0.0) atomicMin(info, (unsigned long long)(goff + kc));
        }
        // ---- 3. swap rows kc and p inside the leaf columns (owners)
        if (p != kc) {
            if (kc >= rbeg && kc < rend && tid < w) slab[tid * chunk + (kc - rbeg)] = s_prow[tid];
            if (p >= rbeg && p < rend && tid < w) slab[tid * chunk + (p - rbeg)] = s_rowk[tid];
        }
        __syncthreads();
        // ---- 4. scale + rank-1 update of own rows > kc; next column's candidate
        bv = -1.0;
        br = LLONG_MAX;
        for (int r = max(0, kc + 1 - rbeg) + tid; r < nr; r += CL_THREADS) {
            const double xk = slab[kk * chunk + r];
            const double l = xk / piv;
            slab[kk * chunk + r] = l;
            double nv = 0.0;
#pragma unroll
            for (int c = 0; c < LEAF_MAX; ++c) {
                const int cc = kk + 1 + c;
                if (cc < w) {
                    const double v = fma(-l, s_prow[cc], slab[cc * chunk + r]);
                    slab[cc * chunk + r] = v;
                    if (c == 0) nv = fabs(v);
                }
            }
            if (kk + 1 < w && better(nv, rbeg + r, bv, br)) { bv = nv; br = rbeg + r; }
        }
        __syncthreads();
    }
    for (int c = 0; c < w; ++c)
        for (int r = tid; r < nr; r += CL_THREADS)
            P[(int64_t)(k0 + c) * ldp + rbeg + r] = slab[c * chunk + r];
    cl.sync();   // no CTA leaves while a peer could still address its shared memory
}


// ---------------------------------------------------------------- gathered FACT (P > 1 tail)
// Combined panel Cp (column-major, ldc): row c = global row j0 + c.  Rows
// c < jb are the replicated top block T; row c >= jb lives on process row
// (g / NB) % P at packed-panel row jb + (g2l(g) - lrL0[p]) of that process's
// panel (column-major, ld ldq[p]), reached through peer memory.
__global__ void fact_gather_kernel(int rows, int jb, int cols, long long j0, int NB, int P,
                                   FactPeers fp, double *Cp, long long ldc)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= rows) return;
    const double *src;
    long long ld;
    if (c < jb) {
        src = fp.panel[fp.myrow] + c;
        ld = fp.ld[fp.myrow];
    } else {
        const long long g = j0 + c;
        const int p = (int)((g / NB) % P);
        const long long l = (g / ((long long)NB * P)) * NB + g % NB;
        src = fp.panel[p] + jb + (l - fp.lrL0[p]);
        ld = fp.ld[p];
    }
    for (int k = blockIdx.y; k < cols; k += gridDim.y) Cp[(long long)k * ldc + c] = __ldcg(src + k * ld);
}

// This process's packed panel [T; own L rows] <- the factored combined panel.
__global__ void fact_extract_kernel(int mine, int jb, int cols, long long j0, int NB, int P,
                                    int myrow, long long lrL0, const double *Cp, long long ldc,
                                    double *Pn, long long ldp)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;   // packed-panel row
    if (r >= jb + mine) return;
    long long c = r;
    if (r >= jb) {
        const long long l = lrL0 + (r - jb);
        const long long g = ((l / NB) * P + myrow) * NB + l % NB;
        c = g - j0;
    }
    for (int k = blockIdx.y; k < cols; k += gridDim.y) Pn[(long long)k * ldp + r] = Cp[(long long)k * ldc + c];
}

constexpr int WARP_LEAF_MIN_ROWS = 128;

// The leaf's CTAs meet at a software grid barrier, so they must be resident
// together: a cooperative launch guarantees that on a GPU with one rank.  In
// the single-device loopback the ranks' leaves also wait on each other, and
// there cooperative launches were measured to stall the device's dispatch
// for seconds now and then (tests/test_loopback.py); the
// loopback caps every leaf grid at SMs / (P*Q) CTAs, so a plain launch is
// co-resident as soon as the (non-waiting) work around it drains.
cudaError_t launch_grid(const FactWork *wk, const void *fn, int G, int NT, void **args,
                        cudaStream_t st)
{
    if (wk->plain_launch) return cudaLaunchKernel(fn, dim3(G), dim3(NT), args, 0, st);
    return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(NT), args, 0, st);
}

void ensure_sms(FactWork *wk)
{
    if (wk->num_sms <= 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&wk->num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (wk->num_sms <= 0) wk->num_sms = 148;
    }
}

cudaError_t cluster_attr()
{
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(leaf_fact_cluster_kernel,
                                        cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (attr_err == cudaSuccess)
            attr_err = cudaFuncSetAttribute(leaf_fact_cluster_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(sizeof(double) * CL_ROWS * LEAF_MAX));
    });
    return attr_err;
}

// grid of the next leaf launch: {CTAs, threads per CTA} from the context's policy
void leaf_grid(const FactWork *wk, int64_t rows, int *G, int *NT)
{
    if (wk->leaf_warp_ctas > 0) {
        *NT = 32;
        *G = (int)std::min<int64_t>(std::max<int64_t>(1, cdiv(rows, WARP_LEAF_MIN_ROWS)),
                                    std::min(wk->leaf_warp_ctas, wk->max_ctas));
        return;
    }
    const int gmax = wk->leaf_max_ctas > 0 ? std::min(wk->leaf_max_ctas, wk->num_sms) : wk->num_sms;
    *NT = FACT_THREADS;
    *G = (int)std::min<int64_t>(std::max<int64_t>(1, cdiv(rows, wk->leaf_rows_per_cta)), gmax);
    *G = std::min(*G, wk->max_ctas);
}

cudaError_t launch_leaf(cudaStream_t st, int64_t m, double *P, int64_t ldp, int k0, int w,
                        int64_t *ipiv, FactWork *wk, long long goff)
{
    ensure_sms(wk);
    unsigned long long *info = reinterpret_cast<unsigned long long *>(wk->info);
    if (wk->leaf_cluster && wk->leaf_variant == 0 && wk->leaf_warp_ctas == 0 &&
        m - k0 <= (int64_t)CL_SIZE * CL_ROWS && w <= LEAF_MAX && w > 0 && m - k0 > 0) {
        const int chunk = (int)cdiv(m - k0, CL_SIZE);
        const size_t smem = sizeof(double) * (size_t)chunk * w;
        cudaError_t e = cluster_attr();
        if (e == cudaSuccess) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(CL_SIZE);
            cfg.blockDim = dim3(CL_THREADS);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = CL_SIZE;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            e = cudaLaunchKernelEx(&cfg, leaf_fact_cluster_kernel, (int)m, ldp, P, k0, w, ipiv,
                                   info, goff, chunk);
        }
        if (e == cudaSuccess) {
            count_launch();
            return cudaSuccess;
        }
        // a device that cannot place a 16-CTA cluster: this context's grid leaf from now on
        cudaGetLastError();
        wk->leaf_cluster = 0;
    }
    int G, NT;
    leaf_grid(wk, m - k0, &G, &NT);
    int m_i = (int)m;
    int64_t ldp_ = ldp;
    int k0_ = k0, w_ = w;
    SpinCtl sc = wk->spin();
    void *args[] = {&m_i, &ldp_, &P, &k0_, &w_, &ipiv, &wk->cand, &wk->bar, &info, &goff, &sc};
    const void *fn = NT == 32 ? (const void *)leaf_fact_kernel<32>
                              : (const void *)leaf_fact_kernel<FACT_THREADS>;
    if (wk->leaf_variant == 1)
        fn = NT == 32 ? (const void *)leaf_fact_ll_kernel<32, false>
                      : (const void *)leaf_fact_ll_kernel<FACT_THREADS, false>;
    else if (wk->leaf_variant == 2)
        fn = NT == 32 ? (const void *)leaf_fact_ll_kernel<32, true>
                      : (const void *)leaf_fact_ll_kernel<FACT_THREADS, true>;
    HPL_CUDA_TRY(launch_grid(wk, fn, G, NT, args, st));
    count_launch();
    return cudaSuccess;
}

cudaError_t launch_leaf_dist(cudaStream_t st, int64_t m, double *P, int64_t ldp, int k0, int w,
                             int64_t *ipiv, FactWork *wk, DistFact *df)
{
    ensure_sms(wk);
    if (df->dp.jbp > 1024) return cudaErrorInvalidValue;
    int G, NT;
    leaf_grid(wk, m, &G, &NT);
    int m_i = (int)m;
    int64_t ldp_ = ldp;
    int k0_ = k0, w_ = w;
    unsigned long long *info = reinterpret_cast<unsigned long long *>(wk->info);
    unsigned long long seq0 = *df->seq;
    unsigned long long *winflag = reinterpret_cast<unsigned long long *>(wk->bar + 8);
    SpinCtl sc = wk->spin();
    void *args[] = {&m_i, &ldp_, &P, &k0_, &w_, &ipiv, &wk->cand, &wk->win, &wk->tsnap,
                    &winflag, &wk->bar, &info, &df->dp, &df->ex, &seq0, &sc};
    const void *fn = NT == 32 ? (const void *)leaf_fact_dist_kernel<32>
                              : (const void *)leaf_fact_dist_kernel<FACT_THREADS>;
    HPL_CUDA_TRY(launch_grid(wk, fn, G, NT, args, st));
    *df->seq += (unsigned long long)w;
    count_launch();
    return cudaSuccess;
}

cudaError_t rec_fact(cudaStream_t st, int64_t m, int64_t nb, double *P, int64_t ldp, int c0,
                     int w, int64_t *ipiv, int nbmin, FactWork *wk, double *scratch,
                     long long goff, DistFact *df)
{
    if (w <= nbmin || w <= 2) {
        if (df) return launch_leaf_dist(st, m, P, ldp, c0, w, ipiv, wk, df);  // full-width swaps
        HPL_CUDA_TRY(launch_leaf(st, m, P, ldp, c0, w, ipiv, wk, goff));
        if (nb > w) {
            panel_laswp_kernel<<<(unsigned)cdiv(nb, 128), 128, 0, st>>>((int)m, (int)nb, ldp, P,
                                                                       c0, w, ipiv);
            count_launch();
            HPL_CUDA_TRY(cudaGetLastError());
        }
        return cudaSuccess;
    }
    // NDIV = 2; the split is rounded down to an even width so
    // every recursion offset stays 16-byte aligned for the TMA operands.
    const int w1 = std::max(2, (w / 2) & ~1), w2 = w - w1;
    HPL_CUDA_TRY(rec_fact(st, m, nb, P, ldp, c0, w1, ipiv, nbmin, wk, scratch, goff, df));
    // U12 <- L11^{-1} U12 (rows c0..c0+w1, cols c0+w1..c0+w)
    HPL_CUDA_TRY(trsm_cols(st, w1, w2, P + (int64_t)c0 * ldp + c0, ldp,
                           P + (int64_t)(c0 + w1) * ldp + c0, ldp, false));
    // A22 -= L21 U12 as the transposed product C'(w2 x m') -= U12^T L21^T:
    // U12^T is repacked col-major into scratch (w2 x w1, ld round16(w2)).
    const int64_t mrest = m - c0 - w1;
    if (mrest > 0) {
        const int64_t lds = round_up(w2, 16);
        HPL_CUDA_TRY(rm_to_cm(st, w2, w1, P + (int64_t)(c0 + w1) * ldp + c0, ldp, scratch, lds));
        HPL_CUDA_TRY(dgemm(st, GEMM_UPDATE, false, w2, mrest, w1, scratch, lds,
                           P + (int64_t)c0 * ldp + c0 + w1, ldp,
                           P + (int64_t)(c0 + w1) * ldp + c0 + w1, ldp, wk->gemm_cfg, nullptr, 0,
                           SLOT_FACT));
    }
    return rec_fact(st, m, nb, P, ldp, c0 + w1, w2, ipiv, nbmin, wk, scratch, goff, df);
}

}  // namespace

cudaError_t fact_prepare()
{
    const cudaError_t e = cluster_attr();
    if (e != cudaSuccess) cudaGetLastError();   // the grid leaf then serves every panel
    return cudaSuccess;
}

void fact_set_leaf_ctas(FactWork *w, int max_ctas, int rows_per_cta)
{
    if (max_ctas >= 0) w->leaf_max_ctas = max_ctas;
    if (rows_per_cta > 0) w->leaf_rows_per_cta = rows_per_cta;
}

cudaError_t fact_work_alloc(FactWork *w)
{
    w->max_ctas = MAX_CTAS;
    w->num_sms = 0;
    w->timeout_ns = 60ull * 1000000000ull;
    HPL_CUDA_TRY(cudaMalloc(&w->cand, sizeof(double) * 2 * (MAX_CTAS + 1) * REC));
    // bar: [0] count, [1] generation, bytes 32..39 the distributed leaf's
    // winner flag, bytes 64..71 the context's abort word (SpinCtl)
    HPL_CUDA_TRY(cudaMalloc(&w->bar, 128));
    HPL_CUDA_TRY(cudaMemset(w->bar, 0, 128));
    w->abort = reinterpret_cast<unsigned long long *>(w->bar + 16);
    HPL_CUDA_TRY(cudaMalloc(&w->info, sizeof(int64_t)));
    HPL_CUDA_TRY(cudaMemset(w->info, 0xff, sizeof(int64_t)));
    HPL_CUDA_TRY(cudaMalloc(&w->win, sizeof(double) * (1024 + 2)));
    HPL_CUDA_TRY(cudaMalloc(&w->tsnap, sizeof(double) * 1024));
    return cudaSuccess;
}

void fact_work_free(FactWork *w)
{
    cudaFree(w->cand);
    cudaFree(w->bar);
    cudaFree(w->info);
    cudaFree(w->win);
    cudaFree(w->tsnap);
    w->win = nullptr;
    w->tsnap = nullptr;
    w->cand = nullptr;
    w->bar = nullptr;
    w->info = nullptr;
    w->abort = nullptr;
}

cudaError_t fact_gather(cudaStream_t st, int64_t rows, int64_t jb, int64_t j0, int NB, int P,
                        const FactPeers &fp, double *Cp, int64_t ldc)
{
    if (rows <= 0) return cudaSuccess;
    dim3 grid((unsigned)cdiv(rows, 256), (unsigned)std::min<int64_t>(jb, 64));
    fact_gather_kernel<<<grid, 256, 0, st>>>((int)rows, (int)jb, (int)jb, j0, NB, P, fp, Cp, ldc);
    count_launch();
    return cudaGetLastError();
}

cudaError_t fact_extract(cudaStream_t st, int64_t mine, int64_t jb, int64_t j0, int NB, int P,
                         int myrow, int64_t lrL0, const double *Cp, int64_t ldc, double *Pn,
                         int64_t ldp)
{
    if (jb + mine <= 0) return cudaSuccess;
    dim3 grid((unsigned)cdiv(jb + mine, 256), (unsigned)std::min<int64_t>(jb, 64));
    fact_extract_kernel<<<grid, 256, 0, st>>>((int)mine, (int)jb, (int)jb, j0, NB, P, myrow, lrL0,
                                              Cp, ldc, Pn, ldp);
    count_launch();
    return cudaGetLastError();
}

cudaError_t panel_fact(cudaStream_t st, int64_t m, int64_t nb, double *P, int64_t ldp,
                       int64_t *ipiv_dev, int nbmin, FactWork *w, double *scratch, int64_t goff,
                       DistFact *dist)
{
    if (nbmin < 1 || nbmin > LEAF_MAX) return cudaErrorInvalidValue;
    if (nb <= 0 || (!dist && m < nb)) return cudaErrorInvalidValue;
    if (m > INT32_MAX) return cudaErrorInvalidValue;
    return rec_fact(st, m, nb, P, ldp, 0, (int)nb, ipiv_dev, nbmin, w, scratch, goff, dist);
}

}  // namespace hpl
