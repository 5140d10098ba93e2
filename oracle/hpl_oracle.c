/*
 * hpl_oracle.c — the CPU ORACLE for the HPL hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path (libhpl.so and the
 * paper_2304_10397_b200 package) never links, imports or calls it, and this
 * file shares no code, header, table or constant generator with the CUDA path.
 *
 * What it computes:
 *   HPL solves A x = b for a dense random FP64 A by LU with partial pivoting
 *   ("based on the open-source HPL implementation"; the phases
 *   FACT/LBCAST/UPDATE/RS).  Blocking, look-ahead, the
 *   2D block-cyclic distribution and the split update are schedule changes
 *   that do not change the mathematics, so this oracle
 *   is the plain DEFINITION: unblocked Gaussian elimination with partial
 *   pivoting (right-looking: pivot search over the column, apply the swap,
 *   then the rank-1 update — PAPER.md l.25), forward and back substitution,
 *   and HPL's scaled residual.  Every loop runs in the textbook order; the
 *   only parallelism is over independent rows, so each element sees the same
 *   operation sequence for any thread count (bitwise thread-count invariant).
 *
 * Compile: gcc -O2 -fopenmp -ffp-contract=off (no FMA contraction, so each
 * a - l*u is a rounded multiply followed by a rounded subtract).
 *
 * Storage: row-major, element (i, j) at A[i*lda + j].
 * Pivot semantics: LAPACK 0-based — ipiv[k] = row swapped with row k at step
 * k ("ipiv[k] is the global row swapped into position k").
 * Tie rule: largest |a|, ties -> smallest row (DESIGN reading A2).
 * Exact zero pivot: stop and report the column (reading A3).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------------------
 * O1. Generator (DESIGN reading A6).  A pure function of
 * (seed, global row, global column) as SPEC.md l.63 requires, indexing the
 * N x (N+1) augmented matrix [A | b] column-major so b = column N never
 * aliases an entry of A.  SplitMix64 finalizer, then an exact map of the top
 * 53 bits onto {k * 2^-53 : -2^52 <= k < 2^52}, a subset of [-0.5, 0.5).
 * ------------------------------------------------------------------------- */
uint64_t oracle_splitmix64(uint64_t seed, uint64_t k)
{
    uint64_t z = seed + (k + 1u) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double oracle_gen_entry(uint64_t seed, int64_t N, int64_t i, int64_t j)
{
    uint64_t k = (uint64_t)j * (uint64_t)N + (uint64_t)i;
    int64_t v = (int64_t)(oracle_splitmix64(seed, k) >> 11) - ((int64_t)1 << 52);
    return ldexp((double)v, -53);
}

/* Fill row-major A (N x N, lda) and b (N) with the seeded HPL system. */
void oracle_generate(uint64_t seed, int64_t N, double *A, int64_t lda, double *b)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        for (int64_t j = 0; j < N; ++j)
            A[i * lda + j] = oracle_gen_entry(seed, N, i, j);
        if (b) b[i] = oracle_gen_entry(seed, N, i, N);
    }
}

/* ---------------------------------------------------------------------------
 * O2. GEPP (LAPACK dgetf2 semantics) on a row-major M x N matrix.
 * For k = 0 .. min(M,N)-1:
 *   p = argmax_{k<=i<M} |A[i][k]|  (first occurrence, i.e. smallest row)
 *   if A[p][k] == 0 -> singular at column k (return k)
 *   ipiv[k] = p; swap rows k and p across all N columns
 *   A[i][k] /= A[k][k]                       for i > k
 *   A[i][c] -= A[i][k] * A[k][c]             for i > k, c > k
 * Returns -1 on success, else the first column with an exact zero pivot.
 * This is also the oracle for a tall-skinny panel FACT (M x NB).
 * ------------------------------------------------------------------------- */
int64_t oracle_getrf(int64_t M, int64_t N, double *A, int64_t lda, int64_t *ipiv)
{
    int64_t kmax = M < N ? M : N;
    for (int64_t k = 0; k < kmax; ++k) {
        int64_t p = k;
        double amax = fabs(A[k * lda + k]);
        for (int64_t i = k + 1; i < M; ++i) {
            double v = fabs(A[i * lda + k]);
            if (v > amax) { amax = v; p = i; }
        }
        ipiv[k] = p;
        if (amax == 0.0) return k;
        if (p != k) {
            double *rk = A + k * lda, *rp = A + p * lda;
            for (int64_t c = 0; c < N; ++c) { double t = rk[c]; rk[c] = rp[c]; rp[c] = t; }
        }
        const double piv = A[k * lda + k];
        const double *rowk = A + k * lda;
#pragma omp parallel for schedule(static)
        for (int64_t i = k + 1; i < M; ++i) {
            double *ri = A + i * lda;
            ri[k] = ri[k] / piv;
            const double l = ri[k];
            for (int64_t c = k + 1; c < N; ++c) ri[c] = ri[c] - l * rowk[c];
        }
    }
    return -1;
}

/* LASWP: apply swaps k = k0 .. k1-1 (rows k <-> ipiv[k]) in order to the
 * columns [c0, c1) of a row-major matrix (the RS phase's row interchanges,
 * PAPER.md l.9 "the row pivots computed in FACT are applied"). */
void oracle_laswp(double *A, int64_t lda, int64_t c0, int64_t c1,
                  int64_t k0, int64_t k1, const int64_t *ipiv)
{
    for (int64_t k = k0; k < k1; ++k) {
        int64_t p = ipiv[k];
        if (p == k) continue;
        for (int64_t c = c0; c < c1; ++c) {
            double t = A[k * lda + c]; A[k * lda + c] = A[p * lda + c]; A[p * lda + c] = t;
        }
    }
}

/* DTRSM of the U block row: B <- L^{-1} B with L (n x n)
 * unit lower triangular, B n x m, both row-major.  Forward substitution,
 * row by row:  B[i][:] -= sum_{k<i} L[i][k] * B[k][:]. */
void oracle_trsm_llnu(int64_t n, int64_t m, const double *L, int64_t ldl,
                      double *B, int64_t ldb)
{
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = 0; k < i; ++k) {
            const double l = L[i * ldl + k];
#pragma omp parallel for schedule(static)
            for (int64_t c = 0; c < m; ++c) B[i * ldb + c] = B[i * ldb + c] - l * B[k * ldb + c];
        }
}

/* Trailing update: C <- C - A * B, C m x n, A m x k,
 * B k x n, all row-major; each C element accumulates its k products in
 * ascending order, then is subtracted once:  C[i][j] - sum_p A[i][p] B[p][j]. */
void oracle_gemm_update(int64_t m, int64_t n, int64_t k,
                        const double *A, int64_t lda, const double *B, int64_t ldb,
                        double *C, int64_t ldc)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (int64_t p = 0; p < k; ++p) s = s + A[i * lda + p] * B[p * ldb + j];
            C[i * ldc + j] = C[i * ldc + j] - s;
        }
}

/* ---------------------------------------------------------------------------
 * O3 / O4. Solve with the factors: apply ipiv to b in order, then
 * L y = P b (unit lower), then U x = y (back substitution).
 * ------------------------------------------------------------------------- */
void oracle_getrs(int64_t N, const double *LU, int64_t lda, const int64_t *ipiv,
                  const double *b, double *x)
{
    double *y = (double *)malloc((size_t)N * sizeof(double));
    memcpy(y, b, (size_t)N * sizeof(double));
    for (int64_t k = 0; k < N; ++k) {
        int64_t p = ipiv[k];
        if (p != k) { double t = y[k]; y[k] = y[p]; y[p] = t; }
    }
    for (int64_t i = 0; i < N; ++i) {
        double s = y[i];
        for (int64_t k = 0; k < i; ++k) s = s - LU[i * lda + k] * y[k];
        y[i] = s;
    }
    for (int64_t i = N - 1; i >= 0; --i) {
        double s = y[i];
        for (int64_t k = i + 1; k < N; ++k) s = s - LU[i * lda + k] * x[k];
        x[i] = s / LU[i * lda + i];
    }
    free(y);
}

/* Back substitution alone: U x = y with U upper (row-major).  Returns -1 or
 * the first (highest) row with an exact zero diagonal. */
int64_t oracle_back_solve(int64_t N, const double *U, int64_t ldu, const double *y, double *x)
{
    for (int64_t i = N - 1; i >= 0; --i) {
        double s = y[i];
        for (int64_t k = i + 1; k < N; ++k) s = s - U[i * ldu + k] * x[k];
        if (U[i * ldu + i] == 0.0) return i;
        x[i] = s / U[i * ldu + i];
    }
    return -1;
}

/* max for the infinity norms: the norm of a vector with a NaN entry is NaN
 * (a plain "v > m" would skip it and a NaN solution would pass the check). */
static double norm_max(double m, double v)
{
    if (m != m || v != v) return NAN;
    return v > m ? v : m;
}

/* ---------------------------------------------------------------------------
 * O5. HPL scaled residual (BASELINE.json north_star):
 *   resid = ||A0 x - b0||_inf / (eps * (||A0||_inf * ||x||_inf + ||b0||_inf) * N)
 * eps = 2^-53 (reading A4), ||A||_inf = max row sum of |a_ij|.  Row sums are
 * accumulated j = 0 .. N-1, then b subtracted.  A0 is given explicitly.
 * Out-params (may be NULL): rinf, anorm, xnorm, bnorm.
 * ------------------------------------------------------------------------- */
double oracle_residual(int64_t N, const double *A0, int64_t lda, const double *x,
                       const double *b0, double *out4)
{
    double rinf = 0.0, anorm = 0.0, xnorm = 0.0, bnorm = 0.0;
    for (int64_t i = 0; i < N; ++i) {
        double s = 0.0, a = 0.0;
        for (int64_t j = 0; j < N; ++j) {
            s = s + A0[i * lda + j] * x[j];
            a = a + fabs(A0[i * lda + j]);
        }
        double r = fabs(s - b0[i]);
        rinf = norm_max(rinf, r);
        anorm = norm_max(anorm, a);
        xnorm = norm_max(xnorm, fabs(x[i]));
        bnorm = norm_max(bnorm, fabs(b0[i]));
    }
    const double eps = ldexp(1.0, -53);
    if (out4) { out4[0] = rinf; out4[1] = anorm; out4[2] = xnorm; out4[3] = bnorm; }
    return rinf / (eps * (anorm * xnorm + bnorm) * (double)N);
}

/* Residual of the seeded system, regenerating A0 and b0 row by row from the
 * generator ("original A, b regenerable from seed"). */
double oracle_residual_seeded(int64_t N, uint64_t seed, const double *x, double *out4)
{
    double rinf = 0.0, anorm = 0.0, xnorm = 0.0, bnorm = 0.0;
#pragma omp parallel
    {
        double lr = 0.0, la = 0.0;
#pragma omp for schedule(static)
        for (int64_t i = 0; i < N; ++i) {
            double s = 0.0, a = 0.0;
            for (int64_t j = 0; j < N; ++j) {
                double v = oracle_gen_entry(seed, N, i, j);
                s = s + v * x[j];
                a = a + fabs(v);
            }
            double r = fabs(s - oracle_gen_entry(seed, N, i, N));
            lr = norm_max(lr, r);
            la = norm_max(la, a);
        }
#pragma omp critical
        {
            rinf = norm_max(rinf, lr);
            anorm = norm_max(anorm, la);
        }
    }
    for (int64_t i = 0; i < N; ++i) {
        xnorm = norm_max(xnorm, fabs(x[i]));
        bnorm = norm_max(bnorm, fabs(oracle_gen_entry(seed, N, i, N)));
    }
    const double eps = ldexp(1.0, -53);
    if (out4) { out4[0] = rinf; out4[1] = anorm; out4[2] = xnorm; out4[3] = bnorm; }
    return rinf / (eps * (anorm * xnorm + bnorm) * (double)N);
}

/* ---------------------------------------------------------------------------
 * The whole oracle run: generate (O1), GEPP (O2), solves (O3/O4), residual
 * (O5).  NB, P, Q do not enter: the oracle is grid-independent by
 * construction.  Returns -1 on success or the singular column.
 * x (N) and ipiv (N) are caller-owned; resid may be NULL.
 * If LU_out is non-NULL (N*N doubles) the row-major factors are copied there.
 * ------------------------------------------------------------------------- */
int64_t oracle_run(int64_t N, uint64_t seed, double *x, int64_t *ipiv, double *resid,
                   double *LU_out)
{
    double *A = (double *)malloc((size_t)N * (size_t)N * sizeof(double));
    double *b = (double *)malloc((size_t)N * sizeof(double));
    if (!A || !b) { free(A); free(b); return -2; }
    oracle_generate(seed, N, A, N, b);
    int64_t info = oracle_getrf(N, N, A, N, ipiv);
    if (info < 0) {
        oracle_getrs(N, A, N, ipiv, b, x);
        if (resid) *resid = oracle_residual_seeded(N, seed, x, NULL);
    }
    if (LU_out) memcpy(LU_out, A, (size_t)N * (size_t)N * sizeof(double));
    free(A); free(b);
    return info;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Pivot maxloc across candidates:
 * the candidate with the largest |value|; ties -> smallest global row.
 * Returns the index into the candidate arrays. */
int64_t oracle_maxloc(int64_t n, const double *absval, const int64_t *row)
{
    int64_t best = 0;
    for (int64_t c = 1; c < n; ++c)
        if (absval[c] > absval[best] || (absval[c] == absval[best] && row[c] < row[best]))
            best = c;
    return best;
}

/* Sampled residual rows at any N (full-size parity):
 * r[t] = sum_j A0[rows[t]][j] * x[j] - b0[rows[t]], j ascending, plus the
 * row sums of |A0| in rsum[t]. */
void oracle_residual_rows(int64_t N, uint64_t seed, const double *x, int64_t nrows,
                          const int64_t *rows, double *r, double *rsum)
{
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < nrows; ++t) {
        const int64_t i = rows[t];
        double s = 0.0, a = 0.0;
        for (int64_t j = 0; j < N; ++j) {
            double v = oracle_gen_entry(seed, N, i, j);
            s = s + v * x[j];
            a = a + fabs(v);
        }
        r[t] = s - oracle_gen_entry(seed, N, i, N);
        rsum[t] = a;
    }
}

/* Thread count for the row-parallel loops (results are thread-count invariant). */
void oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
