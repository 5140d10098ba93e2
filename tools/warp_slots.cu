// warp_slots.cu — which SM sub-partition (SMSP = %warpid mod 4) do the warps
// of co-resident CTAs land on?  The DGEMM (kernels_gemm.cu CfgC) runs 3 CTAs
// of 5 warps per SM (4 DMMA consumer warps + 1 TMA producer); the FP64 pipe
// is per SMSP, so an uneven spread of consumer warps would cap the rate.
// Each warp records (SM, CTA, warp-in-CTA, %warpid) while all CTAs are
// resident (spin 200 us); the host prints consumer warps per SMSP per SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ws tools/warp_slots.cu && /tmp/ws
#include <cuda_runtime.h>
#include <cstdio>
#include <map>
#include <vector>

__global__ void probe(int *out, int consumers)
{
    const int w = threadIdx.x / 32;
    unsigned smid, wid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); while (t - t0 < 200000);
    if ((threadIdx.x & 31) == 0) {
        int *o = out + 4 * (blockIdx.x * (blockDim.x / 32) + w);
        o[0] = (int)smid; o[1] = blockIdx.x; o[2] = w; o[3] = (int)wid;
    }
    (void)consumers;
}

void run(int threads, int ctas_per_sm, int smem, int consumers)
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms * ctas_per_sm, wpc = threads / 32;
    int *d;
    cudaMalloc(&d, sizeof(int) * 4 * grid * wpc);
    probe<<<grid, threads, smem>>>(d, consumers);
    cudaDeviceSynchronize();
    std::vector<int> h(4 * grid * wpc);
    cudaMemcpy(h.data(), d, sizeof(int) * h.size(), cudaMemcpyDeviceToHost);
    cudaFree(d);
    // per SM: consumer warps per SMSP
    std::map<int, std::vector<int>> per;
    for (int i = 0; i < grid * wpc; ++i) {
        const int sm = h[4 * i], w = h[4 * i + 2], wid = h[4 * i + 3];
        auto &v = per[sm];
        v.resize(4);
        if (w < consumers) v[wid % 4]++;
    }
    std::map<std::vector<int>, int> hist;
    for (auto &kv : per) hist[kv.second]++;
    printf("%d threads x %d CTAs/SM (smem %d), consumers = warps 0..%d:\n", threads, ctas_per_sm,
           smem, consumers - 1);
    for (auto &kv : hist)
        printf("   consumers per SMSP {%d %d %d %d}: %d SMs\n", kv.first[0], kv.first[1],
               kv.first[2], kv.first[3], kv.second);
    // first SM's raw slots
    printf("   SM %d warp slots:", h[0]);
    for (int i = 0; i < grid * wpc; ++i)
        if (h[4 * i] == h[0]) printf(" c%d.w%d->%d", h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
    printf("\n");
}

int main()
{
    run(160, 3, 70000, 4);    // CfgC: 3 CTAs of 4 consumers + 1 producer
    run(128, 3, 70000, 4);    // 3 CTAs of 4 warps
    run(160, 2, 100000, 4);   // CfgA-like
    run(288, 2, 100000, 8);   // 2 CTAs of 8 consumers + 1 producer
    run(160, 4, 50000, 4);    // 4 CTAs of 4 consumers + 1 producer
    return 0;
}
