// spin_probe.cu — how many kernels that spin on a flag (one per stream) can
// be resident before a kernel launched on one more stream stops being
// scheduled?  K waiters on K streams, then the setter on stream K+1; a wait
// longer than 200 ms counts as a stall.  Loopback diagnosis.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/sp tools/spin_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void waiter(volatile unsigned long long *flag, unsigned long long want, int *timed_out,
                       int threads_busy)
{
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x != 0) return;
    while (*flag < want) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 200000000ull) {
            atomicAdd(timed_out, 1);
            return;
        }
    }
}
__global__ void setter(volatile unsigned long long *flag, unsigned long long v) { *flag = v; }

int main(int argc, char **argv)
{
    const int maxk = argc > 1 ? atoi(argv[1]) : 64;
    const int threads = argc > 2 ? atoi(argv[2]) : 32;
    std::vector<cudaStream_t> s(maxk + 1);
    for (auto &x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    unsigned long long *flag;
    int *to;
    cudaMalloc(&flag, 8);
    cudaMallocManaged(&to, 4);
    unsigned long long v = 0;
    // warm both kernels
    setter<<<1, 1>>>(flag, 0);
    waiter<<<1, 1>>>(flag, 0, to, 0);
    cudaDeviceSynchronize();
    for (int k = 1; k <= maxk; k *= 2) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(flag, 0, 8);
            *to = 0;
            v = 1;
            cudaDeviceSynchronize();
            for (int i = 0; i < k; ++i) waiter<<<1, threads, 0, s[i]>>>(flag, v, to, 0);
            setter<<<1, 1, 0, s[k]>>>(flag, v);
            cudaDeviceSynchronize();
            printf("K=%d waiters (%d threads each), rep %d: %d timed out\n", k, threads, rep, *to);
        }
    }
    printf("done: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
