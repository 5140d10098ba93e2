/*
 * hpl_kernels.h — kernel-level C ABI of libhpl.so, one entry per row of the
 * hot-path table.  Each call takes HOST buffers, copies them
 * to the device, runs exactly the kernel(s) hpl_factor uses for that step,
 * and copies the result back; the parity tests call these against the CPU
 * oracle.  Not used by hpl_factor itself (which keeps everything in HBM).
 *
 * Return value: 0 on success; otherwise a cudaError_t code (or -1 for an
 * invalid argument, -2 for a singular pivot where noted).  Ownership: all
 * pointers are caller-owned host memory; nothing is retained.
 * Layout legend: "row-major ld" = element (i, j) at p[i*ld + j];
 * "col-major ld" = element (i, j) at p[j*ld + i].
 */
#ifndef HPL_B200_KERNELS_H
#define HPL_B200_KERNELS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* a5/a6 trailing DGEMM (BASELINE north_star "A22 -= L21·U12"):
 * C (m x n, row-major ldc) -= A (m x k, col-major lda) * B (k x n, row-major ldb).
 * Runs the TMA + DMMA kernel.  cfg selects the tile configuration (0: 128x64,
 * 1: 128x128, 2: 64x64; -1 = the default, 2). */
int hplk_dgemm_update(int64_t m, int64_t n, int64_t k,
                      const double *A, int64_t lda, const double *B, int64_t ldb,
                      double *C, int64_t ldc, int32_t cfg);

/* a4 DTRSM of the U block row ("triangular solve on the
 * U-block"): B (k x n, row-major ldb) <- L^{-1} B with L (k x k, col-major
 * ldl) unit lower triangular (upper part and diagonal ignored).  Runs the
 * device path of hpl_factor: unit-lower inverse, then the DMMA kernel. */
int hplk_trsm(int64_t k, int64_t n, const double *L, int64_t ldl, double *B, int64_t ldb);

/* a7 panel FACT: recursive right-looking LU with
 * partial pivoting, NDIV=2, leaf width nbmin, of the m x nb panel P
 * (col-major ldp), in place.  ipiv (nb entries) receives panel-relative
 * LAPACK pivots; the pivot of a column is its max |v| with ties broken
 * towards the smallest row (a8, DESIGN reading A2).  The leaf that picks
 * the pivots is selected like the hpl_set_option knobs of the same names:
 * leaf_variant 0 right-looking / 1 left-looking / 2 Crout (PAPER.md
 * l.27–34), leaf_cluster 1 = the one-cluster shared-memory leaf for panels
 * of <= 16 x 1664 rows (0 = always the cooperative grid leaf), leaf_ctas =
 * grid cap of the grid leaf (0 = all SMs).  *info = -1, or the first column
 * with an exact zero pivot (return -2 then). */
int hplk_panel_fact(int64_t m, int64_t nb, double *P, int64_t ldp, int64_t *ipiv,
                    int32_t nbmin, int32_t leaf_variant, int32_t leaf_cluster, int32_t leaf_ctas,
                    int64_t *info);

/* a1+a3 LASWP gather/scatter ("a GPU kernel to gather the rows
 * ... and a GPU kernel to scatter"): on A (rows x cols, row-major lda), apply
 * the swaps rows (j0+k) <-> ipiv[k], k = 0..jb-1 in order, to columns
 * [c0, c1).  The jb rows that end in block row j0 are gathered into U
 * (jb x (c1-c0), row-major ldu) and NOT written back to A; A receives the
 * displaced rows.  (hpl_factor then writes L11^{-1} U into block row j0.) */
int hplk_laswp(int64_t rows, int64_t cols, double *A, int64_t lda, int64_t j0, int64_t jb,
               const int64_t *ipiv, int64_t c0, int64_t c1, double *U, int64_t ldu);

/* a2+a3 RS (P > 1 row swaps across process rows, PAPER.md l.9 / l.60): the
 * global rows x cols matrix A (row-major lda) is distributed over P process
 * rows block-cyclically (NB-row blocks, block I on process row I mod P), each
 * process row's local rows in their own device buffer — the layout of P
 * ranks, here in one process.  Applies the swaps (j0+k) <-> ipiv[k] (global
 * rows, k < jb, in order) to all columns with the kernels hpl_factor uses:
 * rs_gather_peer on every process row (U = the block's final rows, read from
 * their owners' buffers; W = the original block rows its displaced rows
 * receive), then rs_scatter.  U (jb x cols, row-major ldu) receives process
 * row 0's gathered rows (every process row's U is checked equal: -3 if not);
 * A is updated in place except the block rows j0..j0+jb-1 (which hpl_factor
 * overwrites with the DTRSM result).  j0 must be a multiple of NB. */
int hplk_rs_exchange(int64_t rows, int64_t cols, double *A, int64_t lda, int32_t NB, int32_t P,
                     int64_t j0, int64_t jb, const int64_t *ipiv, double *U, int64_t ldu);

/* a10 back substitution U x = y, U (N x N upper, row-major ldu), block NB. */
int hplk_back_solve(int64_t N, int32_t NB, const double *U, int64_t ldu, const double *y,
                    double *x);

/* a11 generator: out (rows x cols, row-major) = entries (i0+r, j0+c) of the
 * seeded N x (N+1) system (reading A6). */
int hplk_generate(uint64_t seed, int64_t N, int64_t i0, int64_t rows, int64_t j0,
                  int64_t cols, double *out);

/* a11 scaled residual of the seeded system for a given x (N doubles): the
 * kernels hpl_residual runs, on a 1 x 1 grid — A0 and b0 regenerated on the
 * fly from the seed, never stored.  Outputs (host, may be NULL where noted):
 * rsum[i] = sum_j A0[i][j] x[j] (N doubles, may be NULL), asum[i] = sum_j
 * |A0[i][j]| (may be NULL), out4 = {||A0 x - b0||_inf, ||A0||_inf, ||x||_inf,
 * ||b0||_inf} (a non-finite entry reported as +inf), *resid = the scaled
 * residual (+inf if anything is non-finite). */
int hplk_residual(uint64_t seed, int64_t N, const double *x, double *rsum, double *asum,
                  double *out4, double *resid);

/* Measurement hook: time `reps` launches of the trailing-update DGEMM on
 * device-resident operands (m x n x k, generator-filled), CUDA events on the
 * launching stream after one warm-up launch.  ms_out[r] = duration of launch r. */
int hplk_dgemm_bench(int64_t m, int64_t n, int64_t k, int32_t cfg, int32_t reps, double *ms_out);

/* Measurement hook (device analog of PAPER.md Fig. pfact-mptest): time the
 * device panel FACT of an m x nb seeded panel, device-resident, `reps` times
 * (fresh panel each time, CUDA events); leaf_ctas = leaf grid cap (0 = all
 * SMs).  ms_out[r] = duration of rep r.  Returns -2 on a singular panel. */
int hplk_panel_bench(int64_t m, int64_t nb, int32_t nbmin, int32_t leaf_ctas, int32_t reps,
                     double *ms_out);

/* Measurement hook: FP64 tensor-pipe ceiling.  Runs a register-resident chain
 * of mma.sync.m16n8k4.f64 (SASS DMMA) on blocks_per_sm CTAs of `warps` warps
 * per SM; out2 = {ms, flop}. */
int hplk_dmma_peak(int32_t iters, int32_t blocks_per_sm, int32_t warps, double *out2);

#ifdef __cplusplus
}
#endif
#endif /* HPL_B200_KERNELS_H */
