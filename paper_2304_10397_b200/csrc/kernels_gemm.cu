// kernels_gemm.cu — the trailing-update DGEMM (the
// hot loop: "95% of the GPU active time ... inside DGEMM").
//
//   C (m x n, row-major) -= A (m x k, col-major: the packed L panel) * B (k x n,
//   row-major: the U block row)            [GEMM_UPDATE]
//   C = A * B                               [GEMM_ASSIGN, used by the DTRSM]
//
// Design for sm_100a:
//  - FP64 has no tcgen05 kind (ptxas rejects kind::f64), so the tensor-core
//    path is mma.sync.m16n8k4.f64 -> SASS DMMA, accumulators in registers.
//  - Operands are staged by TMA (cp.async.bulk.tensor.2d, 128B swizzle) into a
//    multi-stage shared-memory ring guarded by mbarriers; one producer warp
//    (one elected lane) issues all TMA, the consumer warps only LDS + DMMA.
//  - Fragment layout: MMA rows g / g+8 are mapped to physical rows 2g / 2g+1
//    and the two n8 tiles of a pair to physical columns 2g / 2g+1, so every
//    A and B fragment is ONE 16-byte LDS; the k order inside a 16-deep stage
//    is permuted (k-step s uses rows 8(s>>1)+(s&1)+2t) so that the 128B-swizzle
//    XOR makes those LDS.128 bank-conflict free.  Each thread then owns 2 rows
//    x 4 consecutive columns of C per 16x16 block -> 2x16B global accesses.
//  - Zero-fill of TMA out-of-bounds boxes handles every m/n/k tail.
//  - Tiles are rasterised in groups of GROUP_M m-tiles so the L panel and U
//    block row of a wave stay L2-resident.
#include "hpl_internal.cuh"
#include <type_traits>
#include <cuda.h>
#include <mutex>

namespace hpl {

namespace {

constexpr int BK = 16;         // k-depth of one pipeline stage (4 MMA k-steps)
constexpr int BOX_BYTES = BK * 128;  // one TMA box: BK rows x 16 doubles (128 B)
constexpr int GROUP_M = 16;

struct GemmParams {
    int m, n, k;
    int a_x0, b_x0;            // x offsets of the logical origin inside the tensor maps
    double *C;
    long long ldc;
    double *C2;          // optional second destination (ASSIGN mode only)
    long long ldc2;
    int mode;
    int a_lower;
    int tiles_m, tiles_n;
    int prefetch_c;
    unsigned zero;       // always 0; opaque to the compiler (see release below)
    int ntiles;          // tiles_m * tiles_n; CTA b owns tiles b, b + gridDim.x, ...
    int pair_lower;      // a_lower with even tiles_m: CTA b owns m-tiles i and tiles_m-1-i
};

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_addr(uint32_t addr)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *smem_dst, const CUtensorMap *map, int x, int y,
                                            uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// Explicit shared-space 16-byte load (LDS.128).  A generic load would go
// through the L1TEX path, which the release of the consumer's mbarrier
// arrive does not order against: the next TMA fill could then overwrite the
// stage before the load has read it.
__device__ __forceinline__ double2 lds128(uint32_t addr)
{
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0)
{
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MINB_>
struct Cfg {
    static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
    static constexpr int NWM = BM / WM, NWN = BN / WN, NCW = NWM * NWN;
    static constexpr int THREADS = (NCW + 1) * 32;
    static constexpr int A_BOXES = BM / 16, B_BOXES = BN / 16;
    static constexpr int A_STAGE = A_BOXES * BOX_BYTES, B_STAGE = B_BOXES * BOX_BYTES;
    static constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
    static constexpr int MI = WM / 16, NJ = WN / 16;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8 + 16;
};

// Param-space padding that moves the tensor maps to a role-specific offset.
// Concurrent launches (look-ahead stream vs trailing stream) otherwise place
// their __grid_constant__ tensor maps at the same param-space address, and
// the TMA descriptor cache can then serve one kernel the other's descriptor
// (observed: whole 16-column boxes read from the wrong tensor).
template <int SLOT>
struct alignas(64) ParamPad {
    unsigned char b[64 * (SLOT + 1)];
};

// Epilogue: C -= acc through registers, C prefetched to L2 at tile start.
// (Round 1 measured two alternatives equal and removed them: red.global.add
// of -acc per element, and -acc staged in the drained ring + one TMA
// reduce-add of the tile — DESIGN.md §9.)
template <class C, int SLOT>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
dgemm_tma_kernel(const GemmParams p, const __grid_constant__ ParamPad<SLOT> pad,
                 const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB)
{
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
    uint64_t *empty = full + C::STAGES;

    // ---- grouped rasterisation of the tile grid; several tiles per CTA share
    // one continuous TMA/mbarrier pipeline (the next tile's stages load while
    // the consumers run the current tile's epilogue)
    auto tile_coords = [&](int tile, int &m0, int &n0, int &nk) {
        int pm, pn;
        if (p.pair_lower) {
            // triangular A (the DTRSM's L11^{-1}): m-tile i needs k < 64(i+1),
            // so tile i and its partner tiles_m-1-i together always cost
            // tiles_m+1 tiles of k — every CTA gets the same work
            const int half = p.tiles_m >> 1, G = half * p.tiles_n;
            const bool second = tile >= G;
            const int t = second ? tile - G : tile;
            pn = t / half;
            pm = second ? p.tiles_m - 1 - t % half : t % half;
        } else {
            const int group_sz = GROUP_M * p.tiles_n;
            const int gid = tile / group_sz;
            const int first_m = gid * GROUP_M;
            const int gm = min(p.tiles_m - first_m, GROUP_M);
            pm = first_m + (tile % group_sz) % gm;
            pn = (tile % group_sz) / gm;
        }
        m0 = pm * C::BM;
        n0 = pn * C::BN;
        int k_end = p.k;
        if (p.a_lower) k_end = min(p.k, m0 + C::BM);
        nk = (k_end + BK - 1) / BK;
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == C::NCW) {
        // ================= TMA producer (one lane) =================
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
            int it = 0;
            for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
                int m0, n0, nk;
                tile_coords(tile, m0, n0, nk);
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % C::STAGES;
                    if (it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) & 1) ^ 1);
                    unsigned char *sA = smem + s * C::STAGE_BYTES;
                    unsigned char *sB = sA + C::A_STAGE;
                    mbar_expect_tx(&full[s], C::STAGE_BYTES);
#pragma unroll
                    for (int i = 0; i < C::A_BOXES; ++i)
                        tma_load_2d(sA + i * BOX_BYTES, &tmA, p.a_x0 + m0 + 16 * i, kb * BK, &full[s]);
#pragma unroll
                    for (int i = 0; i < C::B_BOXES; ++i)
                        tma_load_2d(sB + i * BOX_BYTES, &tmB, p.b_x0 + n0 + 16 * i, kb * BK, &full[s]);
                }
            }
        }
        return;
    }

    // ================= consumers =================
    const int wm = warp / C::NWN, wn = warp % C::NWN;
    const int g = lane >> 2, t = lane & 3;
    const int a_box0 = (wm * C::WM) / 16;
    const int b_box0 = (wn * C::WN) / 16;
    const uint32_t smem_base = smem_u32(smem);
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(p.C) & 15) == 0) && ((p.ldc & 1) == 0);
    int it = 0;
    for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    int m0, n0, nk;
    tile_coords(tile, m0, n0, nk);
    const int row_base = m0 + wm * C::WM;   // first row of this warp's tile
    const int col_base = n0 + wn * C::WN;

    if (p.prefetch_c && p.mode == GEMM_UPDATE) {
        // Pull this warp's C tile toward L2 while the mainloop runs: each lane
        // touches the 128-byte lines of its own rows.
        for (int r = lane; r < C::WM; r += 32) {
            const int gr = row_base + r;
            if (gr < p.m) {
                const double *rp = p.C + (long long)gr * p.ldc + col_base;
#pragma unroll
                for (int c = 0; c < C::WN; c += 16)
                    if (col_base + c < p.n)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + c));
            }
        }
    }

    double acc[C::MI][C::NJ][2][4];
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NJ; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[i][j][h][c] = 0.0;

    for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % C::STAGES;
        mbar_wait(&full[s], (it / C::STAGES) & 1);
        // dep folds one word of every fragment loaded from this stage; the
        // release below uses it (masked by a runtime zero) in its address, so
        // the empty-barrier arrive cannot issue before every LDS of the stage
        // has returned.  Without it ptxas places the arrive right after the
        // last LDS is issued, and the next TMA fill can overwrite the stage
        // before that LDS reads it (observed as corrupted 16-column boxes).
        uint32_t dep = 0;
        const uint32_t sA = smem_base + s * C::STAGE_BYTES + a_box0 * BOX_BYTES;
        const uint32_t sB = smem_base + s * C::STAGE_BYTES + C::A_STAGE + b_box0 * BOX_BYTES;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            const int kr = 8 * (ks >> 1) + (ks & 1) + 2 * t;
            const uint32_t off = kr * 128 + ((g ^ (kr & 7)) << 4);
            double2 a[C::MI], b[C::NJ];
#pragma unroll
            for (int i = 0; i < C::MI; ++i) a[i] = lds128(sA + i * BOX_BYTES + off);
#pragma unroll
            for (int j = 0; j < C::NJ; ++j) b[j] = lds128(sB + j * BOX_BYTES + off);
#pragma unroll
            for (int i = 0; i < C::MI; ++i)
                dep ^= __double2loint(a[i].x) ^ __double2loint(a[i].y);
#pragma unroll
            for (int j = 0; j < C::NJ; ++j)
                dep ^= __double2loint(b[j].x) ^ __double2loint(b[j].y);
#pragma unroll
            for (int i = 0; i < C::MI; ++i)
#pragma unroll
                for (int j = 0; j < C::NJ; ++j) {
                    dmma(acc[i][j][0], a[i].x, a[i].y, b[j].x);
                    dmma(acc[i][j][1], a[i].x, a[i].y, b[j].y);
                }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_addr(smem_u32(&empty[s]) + (dep & p.zero));
    }

    // ================= epilogue: C -= acc  (or C = acc) =================
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int row = row_base + 16 * i + 2 * g + h;
            if (row >= p.m) continue;
            double *crow = p.C + (long long)row * p.ldc;
#pragma unroll
            for (int j = 0; j < C::NJ; ++j) {
                const int col = col_base + 16 * j + 4 * t;
                // row 2g: lo.c0 hi.c0 lo.c1 hi.c1 ; row 2g+1: lo.c2 hi.c2 lo.c3 hi.c3
                const double v0 = acc[i][j][0][2 * h], v1 = acc[i][j][1][2 * h];
                const double v2 = acc[i][j][0][2 * h + 1], v3 = acc[i][j][1][2 * h + 1];
                if (vec_ok && col + 3 < p.n) {
                    double2 *q = reinterpret_cast<double2 *>(crow + col);
                    if (p.mode == GEMM_UPDATE) {
                        double2 x0 = q[0], x1 = q[1];
                        x0.x -= v0; x0.y -= v1; x1.x -= v2; x1.y -= v3;
                        q[0] = x0; q[1] = x1;
                    } else {
                        q[0] = make_double2(v0, v1);
                        q[1] = make_double2(v2, v3);
                    }
                } else {
                    const bool upd = p.mode == GEMM_UPDATE;
                    if (col + 0 < p.n) crow[col + 0] = upd ? crow[col + 0] - v0 : v0;
                    if (col + 1 < p.n) crow[col + 1] = upd ? crow[col + 1] - v1 : v1;
                    if (col + 2 < p.n) crow[col + 2] = upd ? crow[col + 2] - v2 : v2;
                    if (col + 3 < p.n) crow[col + 3] = upd ? crow[col + 3] - v3 : v3;
                }
                if (p.C2 != nullptr) {
                    // second copy (16B-aligned by construction, see dgemm())
                    double *c2 = p.C2 + (long long)row * p.ldc2 + col;
                    if (col + 3 < p.n) {
                        reinterpret_cast<double2 *>(c2)[0] = make_double2(v0, v1);
                        reinterpret_cast<double2 *>(c2)[1] = make_double2(v2, v3);
                    } else {
                        if (col + 0 < p.n) c2[0] = v0;
                        if (col + 1 < p.n) c2[1] = v1;
                        if (col + 2 < p.n) c2[2] = v2;
                    }
                }
            }
        }
    }
    }  // tile loop
}

// ---------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                              const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                              const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode()
{
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(f);
    });
    return fn;
}

// 2D map over a matrix whose contiguous dimension has extent xext and whose
// strided dimension (stride ld doubles) has extent yext; box 16 x BK.
cudaError_t make_map(CUtensorMap *map, const double *base, int64_t xext, int64_t yext, int64_t ld)
{
    EncodeFn enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    cuuint64_t gdim[2] = {(cuuint64_t)xext, (cuuint64_t)yext};
    cuuint64_t gstr[1] = {(cuuint64_t)(ld * 8)};
    cuuint32_t box[2] = {16, BK};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), gdim,
                     gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 128x64 tile, 4 consumer warps (64x32 each), 2 CTAs/SM, 4 stages.
using CfgA = Cfg<128, 64, 64, 32, 4, 2>;
// 128x128 tile, 8 consumer warps (64x32 each), 1 CTA/SM, 6 stages.
using CfgB = Cfg<128, 128, 64, 32, 6, 1>;
// 64x64 tile, 4 consumer warps (32x32), 3 CTAs/SM: the default.
// Round 1 measured 6-stage, 4-CTA/SM and 8-warp 64x64 variants slower and
// removed them (profiles/r01_gemm_cfg_probe.log).
using CfgC = Cfg<64, 64, 32, 32, 4, 3>;

template <class C, int SLOT>
cudaError_t set_attr()
{
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(dgemm_tma_kernel<C, SLOT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    });
    return attr_err;
}

template <class C>
cudaError_t set_attr_all()
{
    HPL_CUDA_TRY((set_attr<C, SLOT_TRAIL>()));
    HPL_CUDA_TRY((set_attr<C, SLOT_LOOKAHEAD>()));
    HPL_CUDA_TRY((set_attr<C, SLOT_FACT>()));
    return set_attr<C, SLOT_RS>();
}

template <class C, int SLOT>
cudaError_t launch_slot(cudaStream_t st, const CUtensorMap &ma, const CUtensorMap &mb,
                        const GemmParams &p)
{
    HPL_CUDA_TRY((set_attr<C, SLOT>()));
    ParamPad<SLOT> pad{};
    const unsigned grid = (unsigned)(p.pair_lower ? p.ntiles / 2 : p.ntiles);
    dgemm_tma_kernel<C, SLOT><<<grid, C::THREADS, C::SMEM, st>>>(p, pad, ma, mb);
    count_launch();
    return cudaGetLastError();
}

template <class C>
cudaError_t launch_cfg(cudaStream_t st, const CUtensorMap &ma, const CUtensorMap &mb,
                       GemmParams p, int slot)
{
    p.tiles_m = (int)cdiv(p.m, C::BM);
    p.tiles_n = (int)cdiv(p.n, C::BN);
    p.ntiles = p.tiles_m * p.tiles_n;     // one tile per CTA (two when pair_lower)
    p.pair_lower = p.a_lower && p.tiles_m >= 2 && (p.tiles_m & 1) == 0;
    switch (slot) {
    case SLOT_LOOKAHEAD: return launch_slot<C, SLOT_LOOKAHEAD>(st, ma, mb, p);
    case SLOT_FACT: return launch_slot<C, SLOT_FACT>(st, ma, mb, p);
    case SLOT_RS: return launch_slot<C, SLOT_RS>(st, ma, mb, p);
    default: return launch_slot<C, SLOT_TRAIL>(st, ma, mb, p);
    }
}

}  // namespace

cudaError_t dgemm_prepare()
{
    if (!get_encode()) return cudaErrorNotSupported;
    HPL_CUDA_TRY(set_attr_all<CfgA>());
    HPL_CUDA_TRY(set_attr_all<CfgB>());
    return set_attr_all<CfgC>();
}

cudaError_t dgemm(cudaStream_t st, int mode, bool a_lower, int64_t m, int64_t n, int64_t k,
                  const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                  int64_t ldc, int cfg, double *C2, int64_t ldc2, int slot)
{
    if (C2 && (mode != GEMM_ASSIGN || (reinterpret_cast<uintptr_t>(C2) & 15) || (ldc2 & 1)))
        return cudaErrorInvalidValue;
    if (m <= 0 || n <= 0) return cudaSuccess;
    if (k <= 0) {
        if (mode == GEMM_ASSIGN) {
            return cudaMemset2DAsync(C, ldc * 8, 0, n * 8, m, st);
        }
        return cudaSuccess;
    }
    if ((lda & 1) || (ldb & 1)) return cudaErrorInvalidValue;
    if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) return cudaErrorInvalidValue;
    // TMA boxes must start on 16-byte boundaries under the 128B swizzle (an
    // odd-element start coordinate faults): callers keep A and B aligned.
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
        return cudaErrorMisalignedAddress;
    const double *abase = A, *bbase = B;
    const int ax0 = 0, bx0 = 0;
    CUtensorMap ma, mb;
    HPL_CUDA_TRY(make_map(&ma, abase, ax0 + m, k, lda));
    HPL_CUDA_TRY(make_map(&mb, bbase, bx0 + n, k, ldb));
    GemmParams p{};
    p.m = (int)m; p.n = (int)n; p.k = (int)k;
    p.a_x0 = ax0; p.b_x0 = bx0;
    p.C = C; p.ldc = ldc; p.mode = mode; p.a_lower = a_lower ? 1 : 0;
    p.C2 = C2; p.ldc2 = ldc2;
    p.prefetch_c = 1;
    p.zero = 0;
    if (cfg < 0) cfg = DGEMM_DEFAULT_CFG;
    switch (cfg) {
    case 0: return launch_cfg<CfgA>(st, ma, mb, p, slot);
    case 1: return launch_cfg<CfgB>(st, ma, mb, p, slot);
    case 2: return launch_cfg<CfgC>(st, ma, mb, p, slot);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace hpl
