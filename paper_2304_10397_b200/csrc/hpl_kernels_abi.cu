// hpl_kernels_abi.cu — include/hpl_kernels.h: host-buffer wrappers that run
// exactly the kernels hpl_factor uses for one hot-path step (parity tests).
#include "hpl_internal.cuh"
#include "../../include/hpl_kernels.h"
#include <cstring>
#include <vector>

using namespace hpl;

namespace {

struct Dev {
    void *p = nullptr;
    cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 8); }
    ~Dev() { if (p) cudaFree(p); }
    template <class T> T *as() { return static_cast<T *>(p); }
};

#define KT(expr)                                  \
    do {                                          \
        cudaError_t _e = (expr);                  \
        if (_e != cudaSuccess) return (int)_e;    \
    } while (0)

}  // namespace

extern "C" {

int hplk_dgemm_update(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda,
                      const double *B, int64_t ldb, double *C, int64_t ldc, int32_t cfg)
{
    if (m < 0 || n < 0 || k < 0 || lda < m || ldb < n || ldc < n) return -1;
    // device copies with even (TMA-legal) leading dimensions
    const int64_t dla = round_up(std::max<int64_t>(m, 1), 16), dlb = round_up(std::max<int64_t>(n, 1), 16);
    const int64_t dlc = dlb;
    Dev dA, dB, dC;
    KT(dA.alloc(sizeof(double) * dla * std::max<int64_t>(k, 1)));
    KT(dB.alloc(sizeof(double) * dlb * std::max<int64_t>(k, 1)));
    KT(dC.alloc(sizeof(double) * dlc * std::max<int64_t>(m, 1)));
    if (k > 0 && m > 0)
        KT(cudaMemcpy2D(dA.p, dla * 8, A, lda * 8, m * 8, k, cudaMemcpyHostToDevice));
    if (k > 0 && n > 0)
        KT(cudaMemcpy2D(dB.p, dlb * 8, B, ldb * 8, n * 8, k, cudaMemcpyHostToDevice));
    if (m > 0 && n > 0)
        KT(cudaMemcpy2D(dC.p, dlc * 8, C, ldc * 8, n * 8, m, cudaMemcpyHostToDevice));
    KT(dgemm(0, GEMM_UPDATE, false, m, n, k, dA.as<double>(), dla, dB.as<double>(), dlb,
             dC.as<double>(), dlc, cfg));
    KT(cudaDeviceSynchronize());
    if (m > 0 && n > 0)
        KT(cudaMemcpy2D(C, ldc * 8, dC.p, dlc * 8, n * 8, m, cudaMemcpyDeviceToHost));
    return 0;
}

int hplk_trsm(int64_t k, int64_t n, const double *L, int64_t ldl, double *B, int64_t ldb)
{
    if (k < 0 || n < 0 || ldl < k || ldb < n || k > 1024) return -1;
    if (k == 0 || n == 0) return 0;
    const int64_t dll = round_up(k, 16), dlb = round_up(n, 16);
    Dev dL, dLi, dU, dB;
    KT(dL.alloc(sizeof(double) * dll * k));
    KT(dLi.alloc(sizeof(double) * dll * k));
    KT(dU.alloc(sizeof(double) * dlb * k));
    KT(dB.alloc(sizeof(double) * dlb * k));
    KT(cudaMemcpy2D(dL.p, dll * 8, L, ldl * 8, k * 8, k, cudaMemcpyHostToDevice));
    KT(cudaMemcpy2D(dU.p, dlb * 8, B, ldb * 8, n * 8, k, cudaMemcpyHostToDevice));
    KT(trsm_cols(0, k, k, dL.as<double>(), dll, dLi.as<double>(), dll, true));
    KT(dgemm(0, GEMM_ASSIGN, true, k, n, k, dLi.as<double>(), dll, dU.as<double>(), dlb,
             dB.as<double>(), dlb));
    KT(cudaDeviceSynchronize());
    KT(cudaMemcpy2D(B, ldb * 8, dB.p, dlb * 8, n * 8, k, cudaMemcpyDeviceToHost));
    return 0;
}

int hplk_panel_fact(int64_t m, int64_t nb, double *P, int64_t ldp, int64_t *ipiv, int32_t nbmin,
                    int32_t leaf_variant, int32_t leaf_cluster, int32_t leaf_ctas, int64_t *info)
{
    if (m < nb || nb < 1 || ldp < m || nbmin < 1 || nbmin > 16) return -1;
    if (leaf_variant < 0 || leaf_variant > 2 || leaf_ctas < 0) return -1;
    const int64_t dlp = round_up(m, 16);
    Dev dP, dI, dS;
    FactWork fw{};
    KT(dP.alloc(sizeof(double) * dlp * nb));
    KT(dI.alloc(sizeof(int64_t) * nb));
    KT(dS.alloc(sizeof(double) * round_up(nb, 16) * nb));
    KT(cudaMemset(dP.p, 0, sizeof(double) * dlp * nb));
    KT(cudaMemcpy2D(dP.p, dlp * 8, P, ldp * 8, m * 8, nb, cudaMemcpyHostToDevice));
    KT(fact_work_alloc(&fw));
    fw.leaf_variant = leaf_variant;
    fw.leaf_cluster = leaf_cluster != 0;
    fact_set_leaf_ctas(&fw, leaf_ctas, 0);
    cudaError_t e = panel_fact(0, m, nb, dP.as<double>(), dlp, dI.as<int64_t>(), nbmin, &fw,
                               dS.as<double>(), 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    int64_t inf = -1;
    if (e == cudaSuccess) e = cudaMemcpy(&inf, fw.info, sizeof inf, cudaMemcpyDeviceToHost);
    fact_work_free(&fw);
    KT(e);
    KT(cudaMemcpy2D(P, ldp * 8, dP.p, dlp * 8, m * 8, nb, cudaMemcpyDeviceToHost));
    KT(cudaMemcpy(ipiv, dI.p, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost));
    if (info) *info = inf;
    return inf == -1 ? 0 : -2;
}

int hplk_laswp(int64_t rows, int64_t cols, double *A, int64_t lda, int64_t j0, int64_t jb,
               const int64_t *ipiv, int64_t c0, int64_t c1, double *U, int64_t ldu)
{
    if (rows < 0 || cols < 0 || lda < cols || jb < 0 || jb > 1024 || j0 + jb > rows || c0 < 0 ||
        c1 > cols || c1 < c0 || ldu < c1 - c0)
        return -1;
    if (jb == 0) return 0;
    std::vector<int64_t> rel(jb);
    for (int64_t k = 0; k < jb; ++k) {
        if (ipiv[k] < j0 + k || ipiv[k] >= rows) return -1;
        rel[k] = ipiv[k] - j0;
    }
    const int64_t dla = round_up(std::max<int64_t>(cols, 1), 16);
    const int64_t dlu = round_up(std::max<int64_t>(c1 - c0, 1), 16);
    Dev dA, dU, dRel, dG, dSrc, dDisp, dN;
    KT(dA.alloc(sizeof(double) * dla * rows));
    KT(dU.alloc(sizeof(double) * dlu * jb));
    KT(dRel.alloc(sizeof(int64_t) * jb));
    KT(dG.alloc(sizeof(int64_t) * jb));
    KT(dSrc.alloc(sizeof(int64_t) * jb));
    KT(dDisp.alloc(sizeof(int64_t) * 2 * jb));
    KT(dN.alloc(sizeof(int)));
    KT(cudaMemcpy2D(dA.p, dla * 8, A, lda * 8, cols * 8, rows, cudaMemcpyHostToDevice));
    KT(cudaMemcpy(dRel.p, rel.data(), sizeof(int64_t) * jb, cudaMemcpyHostToDevice));
    KT(pivot_plan(0, jb, j0, dRel.as<int64_t>(), j0, rows, dG.as<int64_t>(), dSrc.as<int64_t>(),
                  dDisp.as<int64_t>(), dN.as<int>()));
    KT(laswp_gather_scatter(0, jb, dSrc.as<int64_t>(), dDisp.as<int64_t>(), dN.as<int>(),
                            dA.as<double>(), dla, c0, c1, dU.as<double>(), dlu));
    KT(cudaDeviceSynchronize());
    KT(cudaMemcpy2D(A, lda * 8, dA.p, dla * 8, cols * 8, rows, cudaMemcpyDeviceToHost));
    if (c1 > c0)
        KT(cudaMemcpy2D(U, ldu * 8, dU.p, dlu * 8, (c1 - c0) * 8, jb, cudaMemcpyDeviceToHost));
    return 0;
}

int hplk_rs_exchange(int64_t rows, int64_t cols, double *A, int64_t lda, int32_t NB, int32_t P,
                     int64_t j0, int64_t jb, const int64_t *ipiv, double *U, int64_t ldu)
{
    if (rows < 1 || cols < 1 || lda < cols || NB < 1 || P < 1 || P > MAX_P || jb < 1 ||
        jb > 1024 || j0 % NB || j0 + jb > rows || ldu < cols)
        return -1;
    std::vector<int64_t> rel(jb);
    for (int64_t k = 0; k < jb; ++k) {
        if (ipiv[k] < j0 + k || ipiv[k] >= rows) return -1;
        rel[k] = ipiv[k] - j0;
    }
    // process row p's local rows: global rows g with (g / NB) % P == p, in order
    const int64_t ld = round_up(cols, 16);
    std::vector<Dev> dA(P), dU(P), dW(P);
    std::vector<int64_t> mloc(P);
    RsPeers pr{};
    pr.P = P;
    for (int p = 0; p < P; ++p) {
        int64_t m = 0;
        for (int64_t g = 0; g < rows; ++g) m += (g / NB) % P == p;
        mloc[p] = m;
        KT(dA[p].alloc(sizeof(double) * ld * std::max<int64_t>(m, 1)));
        KT(dU[p].alloc(sizeof(double) * ld * jb));
        KT(dW[p].alloc(sizeof(double) * ld * jb));
        int64_t l = 0;
        for (int64_t g = 0; g < rows; ++g)
            if ((g / NB) % P == p)
                KT(cudaMemcpy(dA[p].as<double>() + (l++) * ld, A + g * lda, cols * 8,
                              cudaMemcpyHostToDevice));
        pr.A[p] = dA[p].as<double>();
    }
    Dev dRel, dG, dSrc, dDisp, dN;
    KT(dRel.alloc(sizeof(int64_t) * jb));
    KT(dG.alloc(sizeof(int64_t) * jb));
    KT(dSrc.alloc(sizeof(int64_t) * jb));
    KT(dDisp.alloc(sizeof(int64_t) * 2 * jb));
    KT(dN.alloc(sizeof(int)));
    KT(cudaMemcpy(dRel.p, rel.data(), sizeof(int64_t) * jb, cudaMemcpyHostToDevice));
    KT(pivot_plan(0, jb, j0, dRel.as<int64_t>(), j0, rows, dG.as<int64_t>(), dSrc.as<int64_t>(),
                  dDisp.as<int64_t>(), dN.as<int>()));
    // phase 1 on every process row (the peers' A read in place), then phase 2
    // — the order the two flag barriers of rs_cols enforce
    for (int p = 0; p < P; ++p) {
        pr.myrow = p;
        KT(rs_gather_peer(0, jb, dSrc.as<int64_t>(), dDisp.as<int64_t>(), dN.as<int>(), pr, ld, 0,
                          cols, dU[p].as<double>(), ld, dW[p].as<double>(), ld, j0, NB));
    }
    for (int p = 0; p < P; ++p)
        KT(rs_scatter(0, dDisp.as<int64_t>(), dN.as<int>(), dW[p].as<double>(), ld, j0,
                      dA[p].as<double>(), ld, 0, cols, NB, P, p));
    KT(cudaDeviceSynchronize());
    for (int p = 0; p < P; ++p) {
        int64_t l = 0;
        for (int64_t g = 0; g < rows; ++g)
            if ((g / NB) % P == p)
                KT(cudaMemcpy(A + g * lda, dA[p].as<double>() + (l++) * ld, cols * 8,
                              cudaMemcpyDeviceToHost));
    }
    // every process row gathered the same U: return process row 0's, check the rest
    KT(cudaMemcpy2D(U, ldu * 8, dU[0].p, ld * 8, cols * 8, jb, cudaMemcpyDeviceToHost));
    std::vector<double> other((size_t)cols * jb);
    for (int p = 1; p < P; ++p) {
        KT(cudaMemcpy2D(other.data(), cols * 8, dU[p].p, ld * 8, cols * 8, jb,
                        cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < jb; ++k)
            if (std::memcmp(other.data() + k * cols, U + k * ldu, cols * 8)) return -3;
    }
    return 0;
}

int hplk_back_solve(int64_t N, int32_t NB, const double *U, int64_t ldu, const double *y,
                    double *x)
{
    if (N < 1 || NB < 1 || NB > 1024 || ldu < N) return -1;
    const int64_t dl = round_up(N + 1, 16);
    Dev dU, dX, dT;
    KT(dU.alloc(sizeof(double) * dl * N));
    KT(dX.alloc(sizeof(double) * N));
    KT(dT.alloc(sizeof(double) * 2 * 17 * NB));
    KT(cudaMemcpy2D(dU.p, dl * 8, U, ldu * 8, N * 8, N, cudaMemcpyHostToDevice));
    // y goes into column N (the layout hpl_solve sees)
    KT(cudaMemcpy2D(dU.as<double>() + N, dl * 8, y, 8, 8, N, cudaMemcpyHostToDevice));
    KT(back_solve(0, N, NB, dU.as<double>(), dl, dU.as<double>() + N, dl, dX.as<double>(),
                  dT.as<double>()));
    KT(cudaDeviceSynchronize());
    KT(cudaMemcpy(x, dX.p, sizeof(double) * N, cudaMemcpyDeviceToHost));
    return 0;
}

int hplk_generate(uint64_t seed, int64_t N, int64_t i0, int64_t rows, int64_t j0, int64_t cols,
                  double *out)
{
    if (N < 1 || rows < 0 || cols < 0 || i0 < 0 || j0 < 0 || i0 + rows > N || j0 + cols > N + 1)
        return -1;
    if (rows == 0 || cols == 0) return 0;
    Dev d;
    KT(d.alloc(sizeof(double) * rows * cols));
    KT(gen_window(0, seed, N, i0, rows, j0, cols, d.as<double>(), cols));
    KT(cudaDeviceSynchronize());
    KT(cudaMemcpy(out, d.p, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost));
    return 0;
}

int hplk_residual(uint64_t seed, int64_t N, const double *x, double *rsum, double *asum,
                  double *out4, double *resid)
{
    if (N < 1 || !x || !out4 || !resid) return -1;
    Dev dx, dr, da, d4;
    KT(dx.alloc(sizeof(double) * N));
    KT(dr.alloc(sizeof(double) * N));
    KT(da.alloc(sizeof(double) * N));
    KT(d4.alloc(sizeof(double) * 4));
    KT(cudaMemcpy(dx.p, x, sizeof(double) * N, cudaMemcpyHostToDevice));
    // the kernels hpl_residual runs on a 1 x 1 grid (block-cyclic map = identity)
    KT(residual_partial(0, seed, N, 1, 1, 0, N, 1, 0, N, dx.as<double>(), dr.as<double>(),
                        da.as<double>()));
    KT(residual_finalize(0, seed, N, 1, 1, 0, N, dr.as<double>(), da.as<double>(),
                         dx.as<double>(), d4.as<double>()));
    KT(cudaDeviceSynchronize());
    if (rsum) KT(cudaMemcpy(rsum, dr.p, sizeof(double) * N, cudaMemcpyDeviceToHost));
    if (asum) KT(cudaMemcpy(asum, da.p, sizeof(double) * N, cudaMemcpyDeviceToHost));
    KT(cudaMemcpy(out4, d4.p, sizeof(double) * 4, cudaMemcpyDeviceToHost));
    *resid = scaled_residual(out4, N);
    return 0;
}

int hplk_dgemm_bench(int64_t m, int64_t n, int64_t k, int32_t cfg, int32_t reps, double *ms_out)
{
    if (m < 1 || n < 1 || k < 1 || reps < 1 || !ms_out || cfg < -1 || cfg > 2) return -1;
    const int64_t lda = round_up(m, 16), ldb = round_up(n, 16), ldc = ldb;
    Dev dA, dB, dC;
    KT(dA.alloc(sizeof(double) * lda * k));
    KT(dB.alloc(sizeof(double) * ldb * k));
    KT(dC.alloc(sizeof(double) * ldc * m));
    KT(gen_window(0, 1, lda, 0, k, 0, lda, dA.as<double>(), lda));
    KT(gen_window(0, 2, ldb, 0, k, 0, ldb, dB.as<double>(), ldb));
    KT(gen_local(0, 3, std::max(m, ldc), 1 << 20, 1, 1, 0, 0, m, ldc, dC.as<double>(), ldc));
    cudaEvent_t e0, e1;
    KT(cudaEventCreate(&e0));
    KT(cudaEventCreate(&e1));
    KT(dgemm(0, GEMM_UPDATE, false, m, n, k, dA.as<double>(), lda, dB.as<double>(), ldb,
             dC.as<double>(), ldc, cfg));
    for (int r = 0; r < reps; ++r) {
        KT(cudaEventRecord(e0, 0));
        KT(dgemm(0, GEMM_UPDATE, false, m, n, k, dA.as<double>(), lda, dB.as<double>(), ldb,
                 dC.as<double>(), ldc, cfg));
        KT(cudaEventRecord(e1, 0));
        KT(cudaEventSynchronize(e1));
        float ms = 0;
        KT(cudaEventElapsedTime(&ms, e0, e1));
        ms_out[r] = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return 0;
}

int hplk_panel_bench(int64_t m, int64_t nb, int32_t nbmin, int32_t leaf_ctas, int32_t reps,
                     double *ms_out)
{
    if (m < nb || nb < 1 || nb > 1024 || nbmin < 1 || nbmin > 16 || reps < 1 || !ms_out) return -1;
    const int64_t ldp = round_up(m, 16);
    Dev dP, dI, dS;
    FactWork fw{};
    KT(dP.alloc(sizeof(double) * ldp * nb));
    KT(dI.alloc(sizeof(int64_t) * nb));
    KT(dS.alloc(sizeof(double) * round_up(nb, 16) * nb));
    KT(fact_work_alloc(&fw));
    fact_set_leaf_ctas(&fw, leaf_ctas, 512);
    cudaEvent_t e0, e1;
    KT(cudaEventCreate(&e0));
    KT(cudaEventCreate(&e1));
    int64_t inf = -1;
    for (int r = -1; r < reps; ++r) {   // r = -1: warm-up
        // column-major m x nb panel of the seeded HPL system (rows = panel rows)
        KT(gen_local(0, 11 + r, std::max(m, nb) + 1, 1 << 20, 1, 1, 0, 0, nb, ldp, dP.as<double>(),
                     ldp));
        KT(cudaEventRecord(e0, 0));
        KT(panel_fact(0, m, nb, dP.as<double>(), ldp, dI.as<int64_t>(), nbmin, &fw,
                      dS.as<double>(), 0));
        KT(cudaEventRecord(e1, 0));
        KT(cudaEventSynchronize(e1));
        float t = 0;
        KT(cudaEventElapsedTime(&t, e0, e1));
        if (r >= 0) ms_out[r] = t;
    }
    KT(cudaMemcpy(&inf, fw.info, sizeof inf, cudaMemcpyDeviceToHost));
    fact_work_free(&fw);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return inf == -1 ? 0 : -2;
}

int hplk_dmma_peak(int32_t iters, int32_t blocks_per_sm, int32_t warps, double *out2)
{
    if (iters < 10 || blocks_per_sm < 1 || warps < 1 || warps > 32 || !out2) return -1;
    KT(dmma_peak(iters, blocks_per_sm, warps, &out2[0], &out2[1]));
    return 0;
}

}  // extern "C"
