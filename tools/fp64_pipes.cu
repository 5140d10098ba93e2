// fp64_pipes.cu — are the FP64 tensor pipe (DMMA, mma.sync m16n8k4 f64) and
// the FP64 FMA pipe (DFMA) separate on sm_100a?  Register-only chains, no
// memory traffic: each CTA runs `wm` warps of DMMA chains and `wf` warps of
// DFMA chains; the rate of each and of the mix is reported.  If the mix beats
// the faster one alone the pipes add up.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64p tools/fp64_pipes.cu
//   /tmp/fp64p
#include <cuda_runtime.h>
#include <cstdio>

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
    return 0;
}
