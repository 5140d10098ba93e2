// fp64_pipes.cu — are the FP64 tensor pipe (DMMA, mma.sync m16n8k4 f64) and
// the FP64 FMA pipe (DFMA) separate on sm_100a?  Register-only chains, no
// memory traffic: each CTA runs `wm` warps of DMMA chains and `wf` warps of
// DFMA chains; the rate of each and of the mix is reported.  If the mix beats
// the faster one alone the pipes add up.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64p tools/fp64_pipes.cu
//   /tmp/fp64p
// Also: the DGEMM consumer loop fed from shared memory (no TMA, no
// epilogue), with and without a register double buffer of the fragments.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0)
{
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

template <int WM, int WF>
__global__ void __launch_bounds__((WM + WF) * 32) pipes(int iters, double *out)
{
    const int w = threadIdx.x / 32;
    double s = 0;
    if (w < WM) {
        double acc[8][4];
        for (int i = 0; i < 8; ++i)
            for (int c = 0; c < 4; ++c) acc[i][c] = 0.0;
        const double a0 = threadIdx.x * 1e-9, a1 = 1e-9, b0 = 1.0 + 1e-12;
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(acc[i], a0, a1, b0);
        for (int i = 0; i < 8; ++i)
            for (int c = 0; c < 4; ++c) s += acc[i][c];
    } else {
        double x[16];
        for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
        const double m = 1.0 - 1e-12, a = 1e-13;
        // one DMMA = 1024 flop per warp = 16 DFMA per thread; 8 DMMA per
        // iteration -> 128 DFMA per thread per iteration for the same flop
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int i = 0; i < 16; ++i) x[i] = fma(x[i], m, a);
        for (int i = 0; i < 16; ++i) s += x[i];
    }
    if (s == 12345.678) out[0] = s;
}

// The DGEMM consumer warp's inner loop (kernels_gemm.cu, CfgC 32x32 warp
// tile): per k-step 2 A + 2 B fragments by ld.shared.v2.f64 from a swizzled
// 128-B-row stage, then 8 m16n8k4 DMMAs; PREF=1 loads the next k-step's
// fragments before the current DMMAs (register double buffer).
__device__ __forceinline__ double2 lds128(uint32_t addr)
{
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
    return v;
}

template <int PREF>
__global__ void __launch_bounds__(128, 4) ldsfed(int iters, double *out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x)
        reinterpret_cast<double *>(sm)[i] = 1e-9 * i;
    __syncthreads();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
    const uint32_t sA = base + (w & 1) * 2 * 2048, sB = base + 16384 + (w >> 1) * 2 * 2048;
    double acc[2][2][2][4] = {};
    auto offs = [&](int ks) {
        const int kr = 8 * (ks >> 1) + (ks & 1) + 2 * t;
        return (uint32_t)(kr * 128 + ((g ^ (kr & 7)) << 4));
    };
    for (int it = 0; it < iters; ++it) {
        if (PREF) {
            double2 a[2], b[2], an[2], bn[2];
            uint32_t off = offs(0);
            for (int i = 0; i < 2; ++i) a[i] = lds128(sA + i * 2048 + off);
            for (int j = 0; j < 2; ++j) b[j] = lds128(sB + j * 2048 + off);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                if (ks < 3) {
                    off = offs(ks + 1);
                    for (int i = 0; i < 2; ++i) an[i] = lds128(sA + i * 2048 + off);
                    for (int j = 0; j < 2; ++j) bn[j] = lds128(sB + j * 2048 + off);
                }
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        dmma(acc[i][j][0], a[i].x, a[i].y, b[j].x);
                        dmma(acc[i][j][1], a[i].x, a[i].y, b[j].y);
                    }
                for (int i = 0; i < 2; ++i) { a[i] = an[i]; b[i] = bn[i]; }
            }
        } else {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint32_t off = offs(ks);
                double2 a[2], b[2];
                for (int i = 0; i < 2; ++i) a[i] = lds128(sA + i * 2048 + off);
                for (int j = 0; j < 2; ++j) b[j] = lds128(sB + j * 2048 + off);
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        dmma(acc[i][j][0], a[i].x, a[i].y, b[j].x);
                        dmma(acc[i][j][1], a[i].x, a[i].y, b[j].y);
                    }
            }
        }
    }
    double s = 0;
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            for (int h = 0; h < 2; ++h)
                for (int c = 0; c < 4; ++c) s += acc[i][j][h][c];
    if (s == 12345.678) out[0] = s;
}

template <int PREF>
void run_lds(const char *name, int blocks_per_sm, int sms, int iters, double *out)
{
    cudaFuncSetAttribute(ldsfed<PREF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * blocks_per_sm;
    ldsfed<PREF><<<grid, 128, 32768>>>(iters, out);
    cudaEventRecord(e0);
    ldsfed<PREF><<<grid, 128, 32768>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 1024.0 * 32 * (double)iters * 4 * grid;
    printf("%-28s blocks/SM %d: %.2f TF/s (%.2f ms) %s\n", name, blocks_per_sm, flop / ms / 1e9, ms,
           cudaGetErrorString(cudaGetLastError()));
}

template <int WM, int WF>
void run(const char *name, int blocks_per_sm, int sms, int iters, double *out)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * blocks_per_sm;
    pipes<WM, WF><<<grid, (WM + WF) * 32>>>(iters, out);
    cudaEventRecord(e0);
    pipes<WM, WF><<<grid, (WM + WF) * 32>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // per DMMA: 16x8x4 MACs = 512 FMA = 1024 flop; per DFMA thread-op: 2 flop
    const double flop_m = 1024.0 * 8 * (double)iters * WM * grid;
    const double flop_f = 2.0 * 16 * 8 * (double)iters * 32 * WF * grid;
    printf("%-28s blocks/SM %d: DMMA %.2f TF/s  DFMA %.2f TF/s  total %.2f TF/s  (%.2f ms) %s\n", name,
           blocks_per_sm, flop_m / ms / 1e9, flop_f / ms / 1e9, (flop_m + flop_f) / ms / 1e9, ms,
           cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 8);
    const int it = 20000;
    run<8, 0>("DMMA only (8 warps)", 2, sms, it, out);
    run<0, 8>("DFMA only (8 warps)", 2, sms, it, out);
    run<8, 8>("DMMA 8 + DFMA 8 warps", 2, sms, it, out);
    run<8, 4>("DMMA 8 + DFMA 4 warps", 2, sms, it, out);
    run<12, 4>("DMMA 12 + DFMA 4 warps", 1, sms, it, out);
    run<4, 4>("DMMA 4 + DFMA 4 warps", 2, sms, it, out);
    run<4, 0>("DMMA only (4 warps)", 3, sms, it, out);
    run<4, 0>("DMMA only (4 warps)", 2, sms, it, out);
    run_lds<0>("LDS-fed 4 warps", 3, sms, it / 4, out);
    run_lds<1>("LDS-fed 4 warps, prefetch", 3, sms, it / 4, out);
    run_lds<0>("LDS-fed 4 warps", 4, sms, it / 4, out);
    run_lds<1>("LDS-fed 4 warps, prefetch", 4, sms, it / 4, out);
    return 0;
}
