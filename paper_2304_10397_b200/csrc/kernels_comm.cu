// kernels_comm.cu — the peer-memory collectives of the non-hot exchanges
// (hpl_internal.cuh "peer collectives"): the replicated top block of the
// P > 1 FACT, the back-solve reductions / broadcasts, the residual norms and
// the singular-column minimum (SPEC.md l.205–213 and l.374–391 name these
// exchanges; the hot-path RS / LBCAST / pivot search have their own kernels).
//
// A collective is: stage -> group_barrier -> read every member's stage in a
// fixed member order -> group_barrier.  Both kernels are tiny; the staging
// copies are copy-engine memcpys.  Every wait is bounded (SpinCtl).
#include "hpl_internal.cuh"

namespace hpl {

namespace {

// lane m < size: announce arrival to member m, then wait for member m's arrival.
__global__ void group_barrier_kernel(GroupDev g, unsigned long long value, SpinCtl sc)
{
    const int m = threadIdx.x;
    if (m >= g.size) return;
    __threadfence_system();
    st_release_sys(&g.blk[m]->flag[g.gid][g.me], value);
    spin_geq_sys(&g.blk[g.me]->flag[g.gid][m], value, sc,
                 SITE_GROUP_BARRIER | (unsigned long long)g.gid << 4 | (unsigned long long)m << 8);
    __threadfence_system();
}

// NaN-propagating max (fmax drops NaN operands: a NaN residual must not
// vanish from the norm).
__device__ __forceinline__ double max_nan(double a, double b)
{
    if (a != a) return a;
    if (b != b) return b;
    return a > b ? a : b;
}

template <int OP>
__global__ void group_reduce_kernel(GroupDev g, long long n, void *out)
{
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
        if (OP == COLL_MIN_U64) {
            unsigned long long v = __ldcg(
                reinterpret_cast<const unsigned long long *>(g.blk[0]->stage[g.gid]) + i);
            for (int m = 1; m < g.size; ++m) {
                const unsigned long long w = __ldcg(
                    reinterpret_cast<const unsigned long long *>(g.blk[m]->stage[g.gid]) + i);
                v = w < v ? w : v;
            }
            static_cast<unsigned long long *>(out)[i] = v;
        } else {
            double v = __ldcg(g.blk[0]->stage[g.gid] + i);
            for (int m = 1; m < g.size; ++m) {
                const double w = __ldcg(g.blk[m]->stage[g.gid] + i);
                v = OP == COLL_SUM ? v + w : max_nan(v, w);
            }
            static_cast<double *>(out)[i] = v;
        }
    }
}

// 2D byte copy by SMs (16-byte units when every pitch and base allows it).
__global__ void copy2d_kernel(char *dst, long long dpitch, const char *src, long long spitch,
                              long long width, long long rows, int vec16)
{
    const long long units = vec16 ? width / 16 : width;
    const long long total = units * rows;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += stride) {
        const long long r = i / units, u = i % units;
        if (vec16)
            reinterpret_cast<int4 *>(dst + r * dpitch)[u] =
                __ldcg(reinterpret_cast<const int4 *>(src + r * spitch) + u);
        else
            dst[r * dpitch + u] = src[r * spitch + u];
    }
}

__global__ void fill_u64_kernel(unsigned long long *p, unsigned long long v) { *p = v; }

}  // namespace

cudaError_t copy2d_sm(cudaStream_t st, void *dst, int64_t dpitch, const void *src, int64_t spitch,
                      int64_t width, int64_t rows)
{
    if (width <= 0 || rows <= 0) return cudaSuccess;
    const int vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | dpitch |
                      spitch | width) & 15) == 0;
    const int64_t units = (vec ? width / 16 : width) * rows;
    const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(units, 256), 148 * 4);
    copy2d_kernel<<<blocks, 256, 0, st>>>(static_cast<char *>(dst), dpitch,
                                           static_cast<const char *>(src), spitch, width, rows, vec);
    count_launch();
    return cudaGetLastError();
}

cudaError_t fill_u64(cudaStream_t st, unsigned long long *p, unsigned long long v)
{
    fill_u64_kernel<<<1, 1, 0, st>>>(p, v);
    count_launch();
    return cudaGetLastError();
}

cudaError_t group_barrier(cudaStream_t st, const GroupDev &g, unsigned long long value,
                          const SpinCtl &sc)
{
    if (g.size < 1 || g.size > MAX_GROUP || g.gid < 0 || g.gid >= N_GROUPS)
        return cudaErrorInvalidValue;
    if (g.size == 1) return cudaSuccess;
    group_barrier_kernel<<<1, 32, 0, st>>>(g, value, sc);
    count_launch();
    return cudaGetLastError();
}

cudaError_t group_reduce(cudaStream_t st, const GroupDev &g, int op, int64_t n, void *out)
{
    if (n <= 0) return cudaSuccess;
    if (n > STAGE_DOUBLES) return cudaErrorInvalidValue;
    const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), 296);
    switch (op) {
    case COLL_SUM: group_reduce_kernel<COLL_SUM><<<blocks, 256, 0, st>>>(g, n, out); break;
    case COLL_MAX: group_reduce_kernel<COLL_MAX><<<blocks, 256, 0, st>>>(g, n, out); break;
    case COLL_MIN_U64: group_reduce_kernel<COLL_MIN_U64><<<blocks, 256, 0, st>>>(g, n, out); break;
    default: return cudaErrorInvalidValue;
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace hpl
