// Probe: does TMA reduce-add (cp.reduce.async.bulk.tensor .add) accept FP64
// tensors on sm_100a?  C (64 x 64 doubles, row-major) += S (smem tile).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tma_red_probe tma_red_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k(const __grid_constant__ CUtensorMap tm)
{
    __shared__ __align__(1024) double s[64 * 64];
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) s[i] = -0.5 * i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t a = (uint32_t)__cvta_generic_to_shared(s);
        asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];"
                     ::"l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(0), "r"(a) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main()
{
    double *C;
    cudaMalloc(&C, 64 * 64 * 8);
    double h[64 * 64];
    for (int i = 0; i < 64 * 64; ++i) h[i] = 1.0 + i;
    cudaMemcpy(C, h, sizeof h, cudaMemcpyHostToDevice);
    CUtensorMap tm;
    cuuint64_t gdim[2] = {64, 64};
    cuuint64_t gstr[1] = {64 * 8};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, C, gdim, gstr, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode=%d\n", (int)r);
    k<<<1, 256>>>(tm);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel=%s\n", cudaGetErrorString(e));
    cudaMemcpy(h, C, sizeof h, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 64 * 64; ++i)
        if (h[i] != (1.0 + i) - 0.5 * i) ++bad;
    printf("tma_red_f64 %s (bad=%d, h[5]=%g expect %g)\n", bad ? "WRONG" : "OK", bad, h[5], 1.0 + 5 - 2.5);
    return bad ? 1 : 0;
}
