// queue_probe.cu — do two CUDA streams of one context share a hardware work
// queue (a false dependency)?  For every ordered pair (i, j): stream i gets a
// kernel that waits (bounded) for a flag, then stream j gets the kernel that
// sets it.  If i and j feed the same FIFO the setter cannot start while the
// waiter spins, and the wait times out.  Streams are created like the
// loopback's contexts: per rank s_la (high priority), s_tr (low), s_rs (high).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/qp tools/queue_probe.cu
//   CUDA_DEVICE_MAX_CONNECTIONS=32 /tmp/qp 8
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void waiter(volatile unsigned long long *flag, unsigned long long want, int *timed_out)
{
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (*flag < want) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000ull) {   // 20 ms
            *timed_out = 1;
            return;
        }
    }
}

__global__ void setter(volatile unsigned long long *flag, unsigned long long v) { *flag = v; }

int main(int argc, char **argv)
{
    const int ranks = argc > 1 ? atoi(argv[1]) : 8;
    const char *mc = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    std::vector<cudaStream_t> s;
    std::vector<const char *> role;
    for (int r = 0; r < ranks; ++r) {
        cudaStream_t a, b, c;
        cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, hi);
        cudaStreamCreateWithPriority(&b, cudaStreamNonBlocking, lo);
        cudaStreamCreateWithPriority(&c, cudaStreamNonBlocking, hi);
        s.push_back(a); role.push_back("la");
        s.push_back(b); role.push_back("tr");
        s.push_back(c); role.push_back("rs");
    }
    unsigned long long *flag;
    int *to;
    cudaMalloc(&flag, 8);
    cudaMallocManaged(&to, 4);
    cudaMemset(flag, 0, 8);
    unsigned long long v = 0;
    int bad = 0;
    const int n = (int)s.size();
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            if (i == j) continue;
            *to = 0;
            ++v;
            waiter<<<1, 1, 0, s[i]>>>(flag, v, to);
            setter<<<1, 1, 0, s[j]>>>(flag, v);
            cudaDeviceSynchronize();
            if (*to) {
                ++bad;
                printf("false dependency: stream %d (rank %d %s) -> stream %d (rank %d %s)\n", i,
                       i / 3, role[i], j, j / 3, role[j]);
                cudaMemset(flag, 0, 8);   // the setter ran late: reset
                cudaDeviceSynchronize();
                v = 0;
            }
        }
    printf("CUDA_DEVICE_MAX_CONNECTIONS=%s streams=%d pairs=%d false_dependencies=%d (%s)\n",
           mc ? mc : "(unset)", n, n * (n - 1), bad, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
