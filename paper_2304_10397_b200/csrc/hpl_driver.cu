// hpl_driver.cu — the C ABI (include/hpl.h) and the per-iteration schedule.
//
// One iteration j of blocked right-looking LU (SPEC.md glossary l.543–552;
// PAPER.md l.9 for the look-ahead):
//   RS/LASWP(j)  : apply panel j's pivots to the trailing columns (gather the
//                  block row's final rows into U, scatter displaced rows);
//   DTRSM(j)     : block row j <- L11^{-1} U   (L11^{-1} formed once per panel);
//   DGEMM(j)     : A22 -= L21 * U12;
//   FACT(j+1)    : next panel, on the device.
// Look-ahead depth 1 ("perform the UPDATE phase on only the
// leading NB columns, and then immediately begin ... while completing the
// UPDATE phase on the remaining local matrix"): the update of panel j+1's
// columns and FACT(j+1) run on a high-priority stream S_la while the rest of
// the trailing update runs on S_tr; events order the two.
//
// Distribution: 2D block-cyclic over P x Q (rank = p + q*P).
// FACT runs on the process column that owns panel j (P > 1: pivot exchange
// inside the leaf over peer memory, or the gathered FACT for small panels);
// the packed panel (with its pivots) reaches the process row by a copy-engine
// pull over peer memory (LBCAST: "Processes which do not
// participate in the FACT phase simply wait in the LBCAST phase"); the row
// swaps cross process rows as a peer-memory gather (RS).  NCCL carries the
// setup, the replicated top block, the back solve and the residual.
#include "hpl_internal.cuh"
#include "../../include/hpl.h"
#include <nccl.h>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace hpl;

struct hpl_ctx {
    // problem
    int64_t N = 0;
    int NB = 0, P = 1, Q = 1;
    uint64_t seed = 0;
    int rank = 0, nranks = 1, myrow = 0, mycol = 0, device = 0;
    bool dist = false;
    ncclComm_t world = nullptr, row_comm = nullptr, col_comm = nullptr;
    ncclComm_t col_comm_tr = nullptr;            // column comm used only by S_tr (RS of the rest)
    // P > 1: replicated top block, RS buffers (one set per stream), pivot exchange
    double *Tbuf = nullptr;
    double *Ub[3] = {nullptr, nullptr, nullptr}, *Wb[3] = {nullptr, nullptr, nullptr};  // la, right, left
    void *xbuf = nullptr;
    std::vector<void *> xpeer;
    DistExchange xch{};
    unsigned long long xseq = 0;
    // P > 1 RS over peer memory (option rs_peer, default on): every process
    // row's A and barrier flags, IPC-mapped inside the process column
    bool rs_peer = true;
    unsigned long long *rsflag = nullptr;
    std::vector<void *> apeer, fpeer;
    RsPeers rsp{};
    unsigned long long rs_seq[3] = {0, 0, 0};
    // P > 1 gathered panel FACT for small panels (option fact_gather = global
    // rows threshold, 0 = off): the process column's packed panels, mapped
    std::vector<void *> cpeer;
    const double *colpanel[MAX_P][3] = {};
    double *Cp = nullptr;            // combined panel, cp_max_rows x NB (col-major)
    int64_t cp_max_rows = 0;
    int64_t fact_gather_rows = 65536;   // at most this many global rows, and
    double fact_gather_ms = 8.0;        // only where the trailing update is short
                                        // (FACT on the critical path)
    unsigned long long fg_seq = 0;
    // Q > 1 LBCAST over peer memory (option lb_peer, default on): the panel
    // buffers and LBCAST flags of every process column, IPC-mapped inside the
    // process row.  lbflag[o] = last panel (+1) owner o has ready;
    // lbflag[LB_DONE + q] = last panel (+1) of this owner that column q copied.
    static constexpr int LB_DONE = 32;
    bool lb_peer = true;
    unsigned long long lb_base = 0, lb_next = 0;  // flag value of panel j = lb_base + j + 1
    unsigned long long *lbflag = nullptr;
    std::vector<void *> lbpeer;                 // opened handles (Q x (NBUF + 1))
    std::vector<const double *> ppanel;         // [q * NBUF + b]: column q's panel[b]
    std::vector<unsigned long long *> pflag;    // [q]: column q's lbflag
    double *rvec = nullptr, *avec = nullptr;   // residual partial sums (N each)
    // local storage
    int64_t mloc = 0, nloc = 0, lda = 0;
    double *A = nullptr;
    static constexpr int NBUF = 3;   // per-panel state: panels j, j+1, j+2 live at once
    double *panel[NBUF] = {};
    int64_t ldp = 0;
    double *linv[NBUF] = {};
    int64_t ldlinv = 0;
    int64_t *src[NBUF] = {};
    int64_t *disp[NBUF] = {};
    int *ndisp[NBUF] = {};
    int64_t *gpiv = nullptr;
    double *U = nullptr;     // gathered block rows (pre-DTRSM), NB x ldu
    double *U2 = nullptr;    // L11^{-1} U (the DGEMM's B operand), NB x ldu
    int64_t ldu = 0;
    double *scratch = nullptr;
    double *x = nullptr, *tbuf = nullptr, *out4 = nullptr;
    FactWork fw{};
    cudaStream_t s_la = nullptr, s_tr = nullptr;
    cudaStream_t s_la_hi = nullptr, s_la_mid = nullptr;   // s_la is one of these
    cudaEvent_t ev_panel[NBUF] = {}, ev_rest = nullptr;
    cudaEvent_t ev_next = nullptr;   // rest(j) has updated panel j+2's columns
    cudaEvent_t ev_trsm = nullptr;   // rest(j)'s LASWP+DTRSM done: FACT(j+1) may start
    cudaEvent_t ev_trsm0 = nullptr;  // DTRSM of the first column chunk done (trsm_pipe)
    int trsm_pipe = 1;               // DTRSM/DGEMM column chunks of rest(j) (1 = one launch each)
    // split update: RS of one section overlaps the UPDATE of the other
    cudaStream_t s_rs = nullptr;
    cudaEvent_t ev_rsR = nullptr, ev_rsL = nullptr, ev_dgR = nullptr, ev_dgL = nullptr;
    int split_pct = -1;              // right-section share of the local columns; -1 = default
    // options
    bool lookahead = true;
    bool hp_trsm = true;             // rest RS + DTRSM on the high-priority stream
    bool store_l = true;             // write L21 back into A (the solve needs only U and y)
    bool early_next = false;         // (option) update panel j+2's columns first inside rest(j)
    int nbmin = 16;
    bool leaf_auto = true;           // adaptive leaf grid (fact_panel)
    int leaf_few_ctas = 8;
    int leaf_warp = 0;               // >0: hidden FACT uses up to this many one-warp leaf CTAs
    double leaf_hide_ms = 60.0;
    bool timing = false;
    std::vector<cudaEvent_t> tev;   // 7 events per iteration when timing
    std::vector<double> timeline;   // 6 values per iteration (ms)
    std::vector<double> fact_detail;  // 3 values per iteration (ms)
    cudaEvent_t ev_t[3] = {nullptr, nullptr, nullptr};  // factor start/end, solve end
    double factor_ms = 0, solve_ms = 0;
    double dgemm_ms = 0, dgemm_flop = 0;   // trailing (rest) DGEMM launches, timing on
    int64_t dgemm_launches = 0;
    // state
    enum { S_NONE, S_INIT, S_FACTORED, S_SOLVED } state = S_NONE;
    std::string err;
    int64_t singular = -1;
    int64_t launches = 0;
};

namespace {

void set_err(hpl_ctx *c, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
}

#define CK(ctx, expr)                                                                       \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess) {                                                            \
            set_err(ctx, "%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
            return HPL_ERR_CUDA;                                                            \
        }                                                                                   \
    } while (0)

#define NK(ctx, expr)                                                                       \
    do {                                                                                    \
        ncclResult_t _r = (expr);                                                           \
        if (_r != ncclSuccess) {                                                            \
            set_err(ctx, "%s:%d %s -> %s", __FILE__, __LINE__, #expr, ncclGetErrorString(_r)); \
            return HPL_ERR_NCCL;                                                            \
        }                                                                                   \
    } while (0)

// numroc: number of indices of an extent-n dimension owned by coordinate me
int64_t numroc(int64_t n, int nb, int me, int nprocs)
{
    const int64_t nblocks = n / nb;
    int64_t cnt = (nblocks / nprocs) * nb;
    const int64_t extra = nblocks % nprocs;
    if (me < extra) cnt += nb;
    else if (me == extra) cnt += n % nb;
    return cnt;
}

int64_t jb_of(const hpl_ctx *c, int64_t j) { return std::min<int64_t>(c->NB, c->N - j * c->NB); }

// local rows (cols) of this process with global index < g
int64_t lrows_before(const hpl_ctx *c, int64_t g) { return numroc(g, c->NB, c->myrow, c->P); }
int64_t lcols_before(const hpl_ctx *c, int64_t g) { return numroc(g, c->NB, c->mycol, c->Q); }
// Active local rows of iteration j: the block row j (owner process row only)
// starts at local row lr0; the rows below it ("L rows") start at lrL0.
int prow_of(const hpl_ctx *c, int64_t j) { return (int)(j % c->P); }
int64_t lrL0_of(const hpl_ctx *c, int64_t j)
{
    const int64_t lr0 = lrows_before(c, j * c->NB);
    return lr0 + (c->myrow == prow_of(c, j) ? jb_of(c, j) : 0);
}
// The packed panel is [T; L]: T = the jb rows of block row j (replicated on
// the whole process column when P > 1), then this process row's L rows.
int64_t panel_rows(const hpl_ctx *c, int64_t j) { return jb_of(c, j) + (c->mloc - lrL0_of(c, j)); }
int64_t panel_ld(const hpl_ctx *c, int64_t j) { return round_up(panel_rows(c, j), 16); }
int64_t *panel_ipiv(hpl_ctx *c, int64_t j, int b)
{
    // the panel buffer has one extra column; it carries the pivots through LBCAST
    return reinterpret_cast<int64_t *>(c->panel[b] + jb_of(c, j) * panel_ld(c, j));
}

// Packed-panel geometry of process row p for panel j: first local L row,
// number of local L rows, leading dimension of [T; L] (hpl_plan_fact and the
// gathered FACT's peer map use this one function).
void fact_geom(int64_t N, int NB, int P, int p, int64_t j, int64_t *lrL0, int64_t *mL,
               int64_t *ldp)
{
    const int64_t jb = std::min<int64_t>(NB, N - j * NB);
    *lrL0 = numroc(j * NB, NB, p, P) + ((int)(j % P) == p ? jb : 0);
    *mL = numroc(N, NB, p, P) - *lrL0;
    *ldp = round_up(jb + *mL, 16);
}

// P > 1: factor panel j gathered (true) or with the distributed leaf.  Global
// sizes only, so every process of the column takes the same path (the two
// paths issue different peer-memory barriers).
bool use_gathered_fact(int64_t N, int NB, int P, int Q, int64_t j, int64_t gather_rows,
                       double gather_ms, int64_t cp_max_rows)
{
    if (P < 2 || gather_rows <= 0) return false;
    const int64_t rows_total = N - j * NB;   // T + every process row's L rows
    // the per-GPU trailing update this FACT hides behind, at 35 TFLOP/s
    const double rest_ms = 2.0 * (double)cdiv(rows_total, P) * (double)cdiv(rows_total, Q) *
                           (double)NB / 35e12 * 1e3;
    return rows_total <= std::min(gather_rows, cp_max_rows) && rest_ms <= gather_ms;
}

// FACT(j) on the process column that owns panel j: pack [T; L] column-major,
// factor, write the factored panel back to A.
hpl_status fact_local(hpl_ctx *c, cudaStream_t st, int64_t j, int b)
{
    const int64_t j0 = j * c->NB, jb = jb_of(c, j), ldpj = panel_ld(c, j);
    const int64_t lr0 = lrows_before(c, j0), lrL0 = lrL0_of(c, j), mL = c->mloc - lrL0;
    const int64_t lcp = lcols_before(c, j0);
    const bool is_prow = c->myrow == prow_of(c, j);
    if (c->P == 1) {
        // T and L are contiguous local rows [lr0, mloc)
        double *Ablk = c->A + lr0 * c->lda + lcp;
        CK(c, rm_to_cm(st, jb + mL, jb, Ablk, c->lda, c->panel[b], ldpj));
        CK(c, panel_fact(st, jb + mL, jb, c->panel[b], ldpj, panel_ipiv(c, j, b), c->nbmin,
                         &c->fw, c->scratch, j0));
        // write back L11\U11 (U is part of the result); L21 only with store_l
        CK(c, cm_to_rm(st, c->store_l ? jb + mL : jb, jb, c->panel[b], ldpj, Ablk, c->lda));
        return HPL_OK;
    }
    // T from the owner of block row j to the whole process column
    if (is_prow) CK(c, rm_to_cm(st, jb, jb, c->A + lr0 * c->lda + lcp, c->lda, c->Tbuf, jb));
    NK(c, ncclBroadcast(c->Tbuf, c->Tbuf, (size_t)(jb * jb), ncclDouble, prow_of(c, j),
                        c->col_comm, st));
    CK(c, cudaMemcpy2DAsync(c->panel[b], ldpj * 8, c->Tbuf, jb * 8, jb * 8, jb,
                            cudaMemcpyDeviceToDevice, st));
    CK(c, rm_to_cm(st, mL, jb, c->A + lrL0 * c->lda + lcp, c->lda, c->panel[b] + jb, ldpj));
    const int64_t rows_total = c->N - j0;   // T + every process row's L rows
    if (use_gathered_fact(c->N, c->NB, c->P, c->Q, j, c->fact_gather_rows, c->fact_gather_ms,
                          c->cp_max_rows)) {
        // Gathered FACT: barrier (every packed panel of the column is ready),
        // build the combined panel from peer memory, barrier (every peer has
        // read this panel), factor it here (the same arithmetic the
        // distributed leaf performs, so the same bits), keep this process's rows.
        const unsigned long long v = ++c->fg_seq;
        CK(c, rs_barrier(st, c->rsp, 6, v));
        FactPeers fp{};
        fp.myrow = c->myrow;
        for (int p = 0; p < c->P; ++p) {
            int64_t lr0p, mLp, ldq;
            fact_geom(c->N, c->NB, c->P, p, j, &lr0p, &mLp, &ldq);
            fp.panel[p] = c->colpanel[p][b];
            fp.ld[p] = ldq;
            fp.lrL0[p] = lr0p;
        }
        const int64_t ldc = round_up(rows_total, 16);
        CK(c, fact_gather(st, rows_total, jb, j0, c->NB, c->P, fp, c->Cp, ldc));
        CK(c, rs_barrier(st, c->rsp, 7, v));
        if (c->leaf_auto) {
            fact_set_leaf_ctas(0, 512);       // on the critical path: every SM
            fact_set_leaf_warp_ctas(0);
        }
        CK(c, panel_fact(st, rows_total, jb, c->Cp, ldc, panel_ipiv(c, j, b), c->nbmin, &c->fw,
                         c->scratch, j0));
        CK(c, fact_extract(st, mL, jb, j0, c->NB, c->P, c->myrow, lrL0, c->Cp, ldc, c->panel[b],
                           ldpj));
    } else {
    DistFact df{};
    df.dp.j0 = j0; df.dp.lrL0 = lrL0; df.dp.jbp = (int)jb; df.dp.is_prow = is_prow ? 1 : 0;
    df.dp.NB = c->NB; df.dp.P = c->P; df.dp.myrow = c->myrow;
    df.ex = c->xch;
    df.seq = &c->xseq;
    CK(c, panel_fact(st, jb + mL, jb, c->panel[b], ldpj, panel_ipiv(c, j, b), c->nbmin, &c->fw,
                     c->scratch, j0, &df));
    }
    if (c->store_l)
        CK(c, cm_to_rm(st, mL, jb, c->panel[b] + jb, ldpj, c->A + lrL0 * c->lda + lcp, c->lda));
    if (is_prow) CK(c, cm_to_rm(st, jb, jb, c->panel[b], ldpj, c->A + lr0 * c->lda + lcp, c->lda));
    return HPL_OK;
}

// LBCAST(j) along the process row (Q > 1), then on every rank: the pivot
// plan for the row swaps and L11^{-1} for the DTRSM.
hpl_status lbcast_and_plan(hpl_ctx *c, cudaStream_t st, int64_t j, int b)
{
    const int64_t j0 = j * c->NB, jb = jb_of(c, j), ldpj = panel_ld(c, j);
    const int pcol = (int)(j % c->Q);
    const size_t pbytes = sizeof(double) * (size_t)((jb + 1) * ldpj);
    if (c->Q > 1 && c->lb_peer) {
        // owner: announce panel j; receivers: wait for it, pull it with the copy
        // engine over NVLink (no SMs), tell the owner the buffer was read
        FlagOp op{};
        if (c->mycol == pcol) {
            for (int q = 0; q < c->Q; ++q)
                if (q != pcol) op.sig[op.nsig++] = c->pflag[q] + pcol;
            op.sv = c->lb_base + (unsigned long long)j + 1;
            CK(c, flag_op(st, op));
        } else {
            op.wt[op.nwait++] = c->lbflag + pcol;
            op.wv = c->lb_base + (unsigned long long)j + 1;
            CK(c, flag_op(st, op));
            CK(c, cudaMemcpyAsync(c->panel[b], c->ppanel[pcol * hpl_ctx::NBUF + b], pbytes,
                                  cudaMemcpyDeviceToDevice, st));
            FlagOp done{};
            done.sig[done.nsig++] = c->pflag[pcol] + hpl_ctx::LB_DONE + c->mycol;
            done.sv = c->lb_base + (unsigned long long)j + 1;
            CK(c, flag_op(st, done));
        }
    } else if (c->Q > 1) {
        NK(c, ncclBroadcast(c->panel[b], c->panel[b], (size_t)((jb + 1) * ldpj), ncclDouble, pcol,
                            c->row_comm, st));
    }
    // the plan is in GLOBAL rows (P = 1: global == local)
    CK(c, pivot_plan(st, jb, j0, panel_ipiv(c, j, b), j0, c->gpiv + j0, c->src[b], c->disp[b],
                     c->ndisp[b]));
    CK(c, trsm_cols(st, jb, jb, c->panel[b], ldpj, c->linv[b], c->ldlinv, true));
    return HPL_OK;
}

// FACT(j) (owner column) + LBCAST(j) + plan (everyone).
hpl_status fact_panel(hpl_ctx *c, cudaStream_t st, int64_t j, int b, cudaEvent_t ev_pre = nullptr,
                      cudaEvent_t ev_mid = nullptr)
{
    if (ev_pre) CK(c, cudaEventRecord(ev_pre, st));
    if (c->leaf_auto) {
        // The leaf is latency-bound.  While a long trailing DGEMM runs beside it
        // (FACT hidden), a few CTAs leave the SMs to the DGEMM; once the
        // concurrent update is short (FACT on the critical path), use them all.
        const int64_t j0 = j * c->NB, rows = c->mloc - lrows_before(c, j0);
        const int64_t ncols = c->nloc - lcols_before(c, j0);
        const double rest_ms = 2.0 * (double)rows * (double)ncols * c->NB / 35e12 * 1e3;
        // FACT(0) has nothing to hide behind: it always gets every SM
        const bool hide = j > 0 && rest_ms > c->leaf_hide_ms;
        fact_set_leaf_ctas(hide ? c->leaf_few_ctas : 0, 512);
        fact_set_leaf_warp_ctas(hide ? c->leaf_warp : 0);
    }
    if (c->mycol == (int)(j % c->Q)) {
        if (c->Q > 1 && c->lb_peer && j >= c->Q) {
            // panel[b] is about to be overwritten: every other column must have
            // copied this column's previous panel (j - Q) (and so all earlier ones)
            FlagOp op{};
            for (int q = 0; q < c->Q; ++q)
                if (q != c->mycol) op.wt[op.nwait++] = c->lbflag + hpl_ctx::LB_DONE + q;
            op.wv = c->lb_base + (unsigned long long)(j - c->Q) + 1;
            CK(c, flag_op(st, op));
        }
        hpl_status s = fact_local(c, st, j, b);
        if (s != HPL_OK) return s;
    }
    if (ev_mid) CK(c, cudaEventRecord(ev_mid, st));
    return lbcast_and_plan(c, st, j, b);
}

// Column c of the trailing matrix lives at column ucol(c) of the U buffers:
// shifted by one when c is odd so every TMA operand starts 16-byte aligned.
inline int64_t ucol(int64_t c) { return c + (c & 1); }

// Where the RS of a column range left the gathered block rows (U).
struct RsOut {
    double *u = nullptr;
    int64_t ldu = 0;
};
enum { SEC_LA = 0, SEC_RIGHT = 1, SEC_LEFT = 2 };

// RS(j) for local columns [c0, c1): the row interchanges of panel j.  P = 1:
// one local gather/scatter pass; P > 1: across the process column (U = the
// final block rows, each from its owner and summed with zeros elsewhere; W =
// the original block row from its owner, for the displaced rows).
hpl_status rs_cols(hpl_ctx *c, cudaStream_t st, int64_t j, int b, int64_t c0, int64_t c1, int sec,
                   ncclComm_t comm, RsOut *out)
{
    const int64_t j0 = j * c->NB, jb = jb_of(c, j), n = c1 - c0;
    out->u = c->U + ucol(c0);
    out->ldu = c->ldu;
    if (n <= 0) return HPL_OK;
    if (c->P == 1) {
        CK(c, laswp_gather_scatter(st, jb, c->src[b], c->disp[b], c->ndisp[b], jb, c->A, c->lda,
                                   c0, c1, out->u, c->ldu));
        return HPL_OK;
    }
    const int64_t lr0 = lrows_before(c, j0);
    const int64_t ldub = round_up(n, 16);
    double *u = c->Ub[sec], *w = c->Wb[sec];
    if (c->rs_peer) {
        // peer memory: barrier (peers' columns are at iteration j), gather U and
        // this process's W rows over NVLink, barrier (peers done reading), scatter
        const unsigned long long v = ++c->rs_seq[sec];
        CK(c, rs_barrier(st, c->rsp, 2 * sec, v));
        CK(c, rs_gather_peer(st, jb, c->src[b], c->disp[b], c->ndisp[b], c->rsp, c->lda, c0, c1,
                             u, ldub, w, ldub, j0, c->NB));
        CK(c, rs_barrier(st, c->rsp, 2 * sec + 1, v));
        CK(c, rs_scatter(st, c->disp[b], c->ndisp[b], w, ldub, j0, c->A, c->lda, c0, c1, c->NB,
                         c->P, c->myrow));
        out->u = u;
        out->ldu = ldub;
        return HPL_OK;
    }
    CK(c, rs_pack(st, jb, c->src[b], c->A, c->lda, c0, c1, u, ldub, c->NB, c->P, c->myrow));
    if (c->myrow == prow_of(c, j))
        CK(c, cudaMemcpy2DAsync(w, ldub * 8, c->A + lr0 * c->lda + c0, c->lda * 8, n * 8, jb,
                                cudaMemcpyDeviceToDevice, st));
    NK(c, ncclGroupStart());
    NK(c, ncclAllReduce(u, u, (size_t)(jb * ldub), ncclDouble, ncclSum, comm, st));
    NK(c, ncclBroadcast(w, w, (size_t)(jb * ldub), ncclDouble, prow_of(c, j), comm, st));
    NK(c, ncclGroupEnd());
    CK(c, rs_scatter(st, c->disp[b], c->ndisp[b], w, ldub, j0, c->A, c->lda, c0, c1, c->NB, c->P,
                     c->myrow));
    out->u = u;
    out->ldu = ldub;
    return HPL_OK;
}

// DTRSM + DGEMM(j) for local columns [c0, c1) once RS(j) has produced U.
// ev_mid (optional) is recorded between the DTRSM and the DGEMM.
hpl_status compute_cols(hpl_ctx *c, cudaStream_t st, int64_t j, int b, int64_t c0, int64_t c1,
                        const RsOut &rs, cudaEvent_t ev_mid, bool count,
                        cudaEvent_t ev_mid2 = nullptr, bool do_trsm = true, bool do_gemm = true)
{
    const int64_t n = c1 - c0;
    if (n <= 0) {
        if (ev_mid) CK(c, cudaEventRecord(ev_mid, st));
        if (ev_mid2) CK(c, cudaEventRecord(ev_mid2, st));
        return HPL_OK;
    }
    const int slot = st == c->s_la ? SLOT_LOOKAHEAD : SLOT_TRAIL;
    const int64_t j0 = j * c->NB, jb = jb_of(c, j);
    const int64_t lr0 = lrows_before(c, j0), lrL0 = lrL0_of(c, j), ldpj = panel_ld(c, j);
    double *u2 = c->U2 + ucol(c0);
    // block row j <- L11^{-1} U: into U2 (the DGEMM operand) and, on the owner
    // of block row j, into A as well
    if (do_trsm) {
        if (c->myrow == prow_of(c, j))
            CK(c, dgemm(st, GEMM_ASSIGN, true, jb, n, jb, c->linv[b], c->ldlinv, rs.u, rs.ldu,
                        c->A + lr0 * c->lda + c0, c->lda, -1, u2, c->ldu, slot));
        else
            CK(c, dgemm(st, GEMM_ASSIGN, true, jb, n, jb, c->linv[b], c->ldlinv, rs.u, rs.ldu, u2,
                        c->ldu, -1, nullptr, 0, slot));
    }
    if (ev_mid) CK(c, cudaEventRecord(ev_mid, st));
    if (ev_mid2) CK(c, cudaEventRecord(ev_mid2, st));
    const int64_t mrest = c->mloc - lrL0;
    if (mrest > 0 && do_gemm) {
        CK(c, dgemm(st, GEMM_UPDATE, false, mrest, n, jb, c->panel[b] + jb, ldpj, u2, c->ldu,
                    c->A + lrL0 * c->lda + c0, c->lda, -1, nullptr, 0, slot));
        if (count) {
            c->dgemm_flop += 2.0 * (double)mrest * (double)n * (double)jb;
            c->dgemm_launches += 1;
        }
    }
    return HPL_OK;
}

// UPDATE(j) of local columns [c0, c1) on one stream: RS, DTRSM, DGEMM.
// ev (optional, 4 events): recorded before RS, before DTRSM, before DGEMM, after.
hpl_status update_cols(hpl_ctx *c, cudaStream_t st, int64_t j, int b, int64_t c0, int64_t c1,
                       cudaEvent_t *ev = nullptr, cudaEvent_t ev_pre_gemm = nullptr)
{
    if (ev) CK(c, cudaEventRecord(ev[0], st));
    RsOut rs;
    const bool la = st == c->s_la;
    hpl_status s = rs_cols(c, st, j, b, c0, c1, la ? SEC_LA : SEC_RIGHT,
                           la ? c->col_comm : c->col_comm_tr, &rs);
    if (s != HPL_OK) return s;
    if (ev) CK(c, cudaEventRecord(ev[1], st));
    s = compute_cols(c, st, j, b, c0, c1, rs, ev ? ev[2] : nullptr, ev != nullptr, ev_pre_gemm);
    if (s != HPL_OK) return s;
    if (ev) CK(c, cudaEventRecord(ev[3], st));
    return HPL_OK;
}

hpl_status ensure_timing_events(hpl_ctx *c, int64_t nblk)
{
    const size_t need = (size_t)(10 * nblk);
    if (c->tev.size() == need) return HPL_OK;
    for (auto e : c->tev) cudaEventDestroy(e);
    c->tev.assign(need, nullptr);
    for (auto &e : c->tev) CK(c, cudaEventCreate(&e));
    return HPL_OK;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b)
{
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
        cudaGetLastError();
        return 0.f;
    }
    return ms;
}

hpl_status alloc_ctx(hpl_ctx *c)
{
    c->mloc = numroc(c->N, c->NB, c->myrow, c->P);
    c->nloc = numroc(c->N + 1, c->NB, c->mycol, c->Q);
    c->lda = round_up(std::max<int64_t>(c->nloc, 1), 16);
    c->ldp = round_up(std::max<int64_t>(c->mloc + (c->P > 1 ? c->NB : 0), 1), 16);
    c->ldlinv = round_up(c->NB, 16);
    c->ldu = round_up(c->nloc + 2, 16);
    auto M = [&](void **p, size_t bytes) -> bool {
        if (cudaMalloc(p, bytes) != cudaSuccess) {
            cudaGetLastError();
            set_err(c, "cudaMalloc(%zu bytes) failed", bytes);
            return false;
        }
        return true;
    };
    const size_t NBs = (size_t)c->NB;
    if (!M((void **)&c->A, sizeof(double) * (size_t)c->mloc * c->lda)) return HPL_ERR_OOM;
    for (int b = 0; b < hpl_ctx::NBUF; ++b) {
        if (!M((void **)&c->panel[b], sizeof(double) * (size_t)c->ldp * (NBs + 1))) return HPL_ERR_OOM;
        if (!M((void **)&c->linv[b], sizeof(double) * (size_t)c->ldlinv * NBs)) return HPL_ERR_OOM;
        if (!M((void **)&c->src[b], sizeof(int64_t) * NBs)) return HPL_ERR_OOM;
        if (!M((void **)&c->disp[b], sizeof(int64_t) * 2 * NBs)) return HPL_ERR_OOM;
        if (!M((void **)&c->ndisp[b], sizeof(int))) return HPL_ERR_OOM;
        CK(c, cudaMemset(c->panel[b], 0, sizeof(double) * (size_t)c->ldp * (NBs + 1)));
    }
    if (!M((void **)&c->gpiv, sizeof(int64_t) * (size_t)c->N)) return HPL_ERR_OOM;
    if (!M((void **)&c->U, sizeof(double) * NBs * c->ldu)) return HPL_ERR_OOM;
    if (!M((void **)&c->U2, sizeof(double) * NBs * c->ldu)) return HPL_ERR_OOM;
    if (!M((void **)&c->scratch, sizeof(double) * round_up(NBs, 16) * NBs)) return HPL_ERR_OOM;
    if (!M((void **)&c->x, sizeof(double) * (size_t)c->N)) return HPL_ERR_OOM;
    if (!M((void **)&c->tbuf, sizeof(double) * 16 * NBs)) return HPL_ERR_OOM;
    if (!M((void **)&c->out4, sizeof(double) * 4)) return HPL_ERR_OOM;
    if (!M((void **)&c->rvec, sizeof(double) * (size_t)std::max<int64_t>(c->mloc, 1))) return HPL_ERR_OOM;
    if (!M((void **)&c->avec, sizeof(double) * (size_t)std::max<int64_t>(c->mloc, 1))) return HPL_ERR_OOM;
    if (c->P > 1) {
        const size_t rs = sizeof(double) * NBs * (size_t)round_up(c->nloc, 16);
        if (!M((void **)&c->Tbuf, sizeof(double) * NBs * NBs)) return HPL_ERR_OOM;
        for (int k = 0; k < 3; ++k) {
            if (!M((void **)&c->Ub[k], rs)) return HPL_ERR_OOM;
            if (!M((void **)&c->Wb[k], rs)) return HPL_ERR_OOM;
        }
    }
    CK(c, fact_work_alloc(&c->fw));
    int lo, hi;
    CK(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(c, cudaStreamCreateWithPriority(&c->s_la, cudaStreamNonBlocking, hi));
    // the look-ahead stream one level below S_rs (option la_below_rs)
    CK(c, cudaStreamCreateWithPriority(&c->s_la_mid, cudaStreamNonBlocking,
                                       hi < lo ? hi + 1 : hi));
    c->s_la_hi = c->s_la;
    CK(c, cudaStreamCreateWithPriority(&c->s_tr, cudaStreamNonBlocking, lo));
    CK(c, cudaStreamCreateWithPriority(&c->s_rs, cudaStreamNonBlocking, hi));
    for (cudaEvent_t *e : {&c->ev_rsR, &c->ev_rsL, &c->ev_dgR, &c->ev_dgL})
        CK(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (int b = 0; b < hpl_ctx::NBUF; ++b)
        CK(c, cudaEventCreateWithFlags(&c->ev_panel[b], cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&c->ev_next, cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&c->ev_rest, cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&c->ev_trsm, cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&c->ev_trsm0, cudaEventDisableTiming));
    for (int k = 0; k < 3; ++k) CK(c, cudaEventCreate(&c->ev_t[k]));
    return HPL_OK;
}

hpl_status generate(hpl_ctx *c)
{
    CK(c, gen_local(c->s_tr, c->seed, c->N, c->NB, c->P, c->Q, c->myrow, c->mycol, c->mloc,
                    c->nloc, c->A, c->lda));
    CK(c, cudaStreamSynchronize(c->s_tr));
    c->state = hpl_ctx::S_INIT;
    return HPL_OK;
}

void release(hpl_ctx *c)
{
    if (!c) return;
    cudaFree(c->A);
    for (int b = 0; b < hpl_ctx::NBUF; ++b) {
        cudaFree(c->panel[b]); cudaFree(c->linv[b]); 
        cudaFree(c->src[b]); cudaFree(c->disp[b]); cudaFree(c->ndisp[b]);
        if (c->ev_panel[b]) cudaEventDestroy(c->ev_panel[b]);
        if (b == 0 && c->ev_next) cudaEventDestroy(c->ev_next);
    }
    cudaFree(c->gpiv); cudaFree(c->U); cudaFree(c->U2); cudaFree(c->scratch);
    cudaFree(c->x); cudaFree(c->tbuf); cudaFree(c->out4); cudaFree(c->rvec); cudaFree(c->avec);
    cudaFree(c->Tbuf);
    for (int k = 0; k < 3; ++k) { cudaFree(c->Ub[k]); cudaFree(c->Wb[k]); }
    for (void *pp : c->xpeer) if (pp) cudaIpcCloseMemHandle(pp);
    for (void *pp : c->apeer) if (pp) cudaIpcCloseMemHandle(pp);
    for (void *pp : c->cpeer) if (pp) cudaIpcCloseMemHandle(pp);
    cudaFree(c->Cp);
    for (void *pp : c->lbpeer) if (pp) cudaIpcCloseMemHandle(pp);
    cudaFree(c->lbflag);
    for (void *pp : c->fpeer) if (pp) cudaIpcCloseMemHandle(pp);
    cudaFree(c->rsflag);
    cudaFree(c->xbuf);
    if (c->col_comm_tr) ncclCommDestroy(c->col_comm_tr);
    if (c->row_comm) ncclCommDestroy(c->row_comm);
    if (c->col_comm) ncclCommDestroy(c->col_comm);
    if (c->world) ncclCommDestroy(c->world);
    fact_work_free(&c->fw);
    if (c->ev_rest) cudaEventDestroy(c->ev_rest);
    if (c->ev_trsm) cudaEventDestroy(c->ev_trsm);
    if (c->ev_trsm0) cudaEventDestroy(c->ev_trsm0);
    for (cudaEvent_t e : {c->ev_rsR, c->ev_rsL, c->ev_dgR, c->ev_dgL})
        if (e) cudaEventDestroy(e);
    if (c->s_rs) cudaStreamDestroy(c->s_rs);
    for (auto e : c->tev) cudaEventDestroy(e);
    for (int k = 0; k < 3; ++k)
        if (c->ev_t[k]) cudaEventDestroy(c->ev_t[k]);
    if (c->s_la_hi) cudaStreamDestroy(c->s_la_hi);
    if (c->s_la_mid) cudaStreamDestroy(c->s_la_mid);
    if (c->s_tr) cudaStreamDestroy(c->s_tr);
}

// P > 1: pivot-exchange areas shared inside each process column through CUDA
// IPC (peer memory over NVLink); handles travel over the column communicator.
hpl_status setup_exchange(hpl_ctx *c)
{
    const int P = c->P;
    const int recd = 2 + c->NB;
    const size_t rec_bytes = sizeof(double) * 2 * (size_t)P * recd;
    const size_t bytes = rec_bytes + sizeof(unsigned long long) * 2 * P;
    CK(c, cudaMalloc(&c->xbuf, bytes));
    CK(c, cudaMemset(c->xbuf, 0, bytes));
    const size_t fbytes = sizeof(unsigned long long) * RS_SLOTS * MAX_P;
    CK(c, cudaMalloc(&c->rsflag, fbytes));
    CK(c, cudaMemset(c->rsflag, 0, fbytes));
    // six handles per process row: exchange area, local A, RS flags, the
    // three packed-panel buffers (gathered FACT)
    constexpr int NH = 6;
    cudaIpcMemHandle_t h[NH];
    CK(c, cudaIpcGetMemHandle(&h[0], c->xbuf));
    CK(c, cudaIpcGetMemHandle(&h[1], c->A));
    CK(c, cudaIpcGetMemHandle(&h[2], c->rsflag));
    for (int b = 0; b < 3; ++b) CK(c, cudaIpcGetMemHandle(&h[3 + b], c->panel[b]));
    char *dh = nullptr;
    CK(c, cudaMalloc(&dh, sizeof(h) * P));
    CK(c, cudaMemcpy(dh + sizeof(h) * c->myrow, h, sizeof(h), cudaMemcpyHostToDevice));
    NK(c, ncclAllGather(dh + sizeof(h) * c->myrow, dh, sizeof(h), ncclChar, c->col_comm, c->s_la));
    CK(c, cudaStreamSynchronize(c->s_la));
    std::vector<cudaIpcMemHandle_t> hs((size_t)NH * P);
    CK(c, cudaMemcpy(hs.data(), dh, sizeof(h) * P, cudaMemcpyDeviceToHost));
    cudaFree(dh);
    c->xpeer.assign(P, nullptr);
    c->apeer.assign(P, nullptr);
    c->fpeer.assign(P, nullptr);
    c->rsp.P = P;
    c->rsp.myrow = c->myrow;
    c->rsp.my_flag = c->rsflag;
    for (int p = 0; p < P; ++p) {
        if (p == c->myrow) {
            c->rsp.A[p] = c->A;
            c->rsp.flag[p] = c->rsflag;
            for (int b = 0; b < 3; ++b) c->colpanel[p][b] = c->panel[b];
            continue;
        }
        CK(c, cudaIpcOpenMemHandle(&c->apeer[p], hs[NH * p + 1], cudaIpcMemLazyEnablePeerAccess));
        CK(c, cudaIpcOpenMemHandle(&c->fpeer[p], hs[NH * p + 2], cudaIpcMemLazyEnablePeerAccess));
        for (int b = 0; b < 3; ++b) {
            void *ptr = nullptr;
            CK(c, cudaIpcOpenMemHandle(&ptr, hs[NH * p + 3 + b], cudaIpcMemLazyEnablePeerAccess));
            c->cpeer.push_back(ptr);
            c->colpanel[p][b] = static_cast<const double *>(ptr);
        }
        c->rsp.A[p] = static_cast<const double *>(c->apeer[p]);
        c->rsp.flag[p] = static_cast<unsigned long long *>(c->fpeer[p]);
    }
    c->xch.P = P;
    c->xch.myrow = c->myrow;
    c->xch.recd = recd;
    for (int p = 0; p < P; ++p) {
        void *base = c->xbuf;
        if (p != c->myrow) {
            CK(c, cudaIpcOpenMemHandle(&c->xpeer[p], hs[NH * p], cudaIpcMemLazyEnablePeerAccess));
            base = c->xpeer[p];
        }
        c->xch.rec[p] = static_cast<double *>(base);
        c->xch.flag[p] = reinterpret_cast<unsigned long long *>(static_cast<char *>(base) + rec_bytes);
    }
    c->xch.my_rec = c->xch.rec[c->myrow];
    c->xch.my_flag = c->xch.flag[c->myrow];
    // combined panel for the gathered FACT: up to 64 Ki global rows (2^16 x NB doubles)
    c->cp_max_rows = std::min<int64_t>(c->N, (int64_t)1 << 16);
    if (cudaMalloc(&c->Cp, sizeof(double) * (size_t)round_up(c->cp_max_rows, 16) * c->NB) !=
        cudaSuccess) {
        cudaGetLastError();
        set_err(c, "cudaMalloc of the combined panel failed");
        return HPL_ERR_OOM;
    }
    return HPL_OK;
}

// Q > 1: panel buffers + LBCAST flags shared inside each process row (CUDA IPC
// over NVLink); handles travel over the row communicator.  Flags are
// monotonic across factorizations: panel j of a factorization is
// lb_base + j + 1, lb_base advancing past the previous factorization's values.
hpl_status setup_lbcast(hpl_ctx *c)
{
    const int Q = c->Q, NBUF = hpl_ctx::NBUF;
    if (Q > 32) return HPL_ERR_ARG;
    const size_t fbytes = sizeof(unsigned long long) * 64;
    CK(c, cudaMalloc(&c->lbflag, fbytes));
    CK(c, cudaMemset(c->lbflag, 0, fbytes));
    std::vector<cudaIpcMemHandle_t> h(NBUF + 1);
    for (int b = 0; b < NBUF; ++b) CK(c, cudaIpcGetMemHandle(&h[b], c->panel[b]));
    CK(c, cudaIpcGetMemHandle(&h[NBUF], c->lbflag));
    const size_t hb = sizeof(cudaIpcMemHandle_t) * (NBUF + 1);
    char *dh = nullptr;
    CK(c, cudaMalloc(&dh, hb * Q));
    CK(c, cudaMemcpy(dh + hb * c->mycol, h.data(), hb, cudaMemcpyHostToDevice));
    NK(c, ncclAllGather(dh + hb * c->mycol, dh, hb, ncclChar, c->row_comm, c->s_la));
    CK(c, cudaStreamSynchronize(c->s_la));
    std::vector<cudaIpcMemHandle_t> hs((size_t)Q * (NBUF + 1));
    CK(c, cudaMemcpy(hs.data(), dh, hb * Q, cudaMemcpyDeviceToHost));
    cudaFree(dh);
    c->ppanel.assign((size_t)Q * NBUF, nullptr);
    c->pflag.assign(Q, nullptr);
    for (int q = 0; q < Q; ++q) {
        for (int k = 0; k <= NBUF; ++k) {
            void *ptr = nullptr;
            if (q == c->mycol) {
                ptr = k < NBUF ? (void *)c->panel[k] : (void *)c->lbflag;
            } else {
                CK(c, cudaIpcOpenMemHandle(&ptr, hs[(size_t)q * (NBUF + 1) + k],
                                           cudaIpcMemLazyEnablePeerAccess));
                c->lbpeer.push_back(ptr);
            }
            if (k < NBUF) c->ppanel[(size_t)q * NBUF + k] = static_cast<const double *>(ptr);
            else c->pflag[q] = static_cast<unsigned long long *>(ptr);
        }
    }
    return HPL_OK;
}

hpl_status check_args(int64_t N, int32_t NB, int32_t P, int32_t Q)
{
    if (N < 1 || NB < 1 || NB > N || P < 1 || Q < 1) return HPL_ERR_ARG;
    if (NB > 1024) return HPL_ERR_ARG;   // kernel limits (pivot plan, TRSM, back solve)
    if (NB & 1) return HPL_ERR_ARG;      // TMA alignment of the L panel (reading A18)
    if (N >= (int64_t)1 << 31) return HPL_ERR_ARG;
    return HPL_OK;
}

}  // namespace

extern "C" {

hpl_status hpl_init(int64_t N, int32_t NB, int32_t P, int32_t Q, uint64_t seed, hpl_ctx **out)
{
    if (!out) return HPL_ERR_ARG;
    *out = nullptr;
    if (check_args(N, NB, P, Q) != HPL_OK || P * Q != 1) return HPL_ERR_ARG;
    hpl_ctx *c = new hpl_ctx();
    c->N = N; c->NB = NB; c->P = P; c->Q = Q; c->seed = seed;
    cudaGetDevice(&c->device);
    hpl_status s = alloc_ctx(c);
    if (s == HPL_OK) s = generate(c);
    *out = c;   // returned even on failure so hpl_last_error works; caller frees
    return s;
}

hpl_status hpl_init_dist(int64_t N, int32_t NB, int32_t P, int32_t Q, uint64_t seed,
                         int32_t rank, int32_t nranks, const void *nccl_unique_id,
                         int32_t device, hpl_ctx **out)
{
    if (!out || !nccl_unique_id) return HPL_ERR_ARG;
    *out = nullptr;
    if (check_args(N, NB, P, Q) != HPL_OK || P * Q != nranks || rank < 0 || rank >= nranks)
        return HPL_ERR_ARG;
    if (P > MAX_P) return HPL_ERR_ARG;
    hpl_ctx *c = new hpl_ctx();
    *out = c;
    c->N = N; c->NB = NB; c->P = P; c->Q = Q; c->seed = seed;
    c->rank = rank; c->nranks = nranks; c->myrow = rank % P; c->mycol = rank / P;
    c->device = device;
    c->dist = nranks > 1;
    CK(c, cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof id);
    NK(c, ncclCommInitRank(&c->world, nranks, id, rank));
    NK(c, ncclCommSplit(c->world, c->myrow, c->mycol, &c->row_comm, nullptr));
    NK(c, ncclCommSplit(c->world, c->mycol, c->myrow, &c->col_comm, nullptr));
    NK(c, ncclCommSplit(c->world, c->mycol, c->myrow, &c->col_comm_tr, nullptr));
    hpl_status s = alloc_ctx(c);
    if (s == HPL_OK && P > 1) s = setup_exchange(c);
    if (s == HPL_OK && Q > 1) s = setup_lbcast(c);
    if (s == HPL_OK) s = generate(c);
    return s;
}

hpl_status hpl_get_unique_id(void *id_out)
{
    if (!id_out) return HPL_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return HPL_ERR_NCCL;
    std::memcpy(id_out, &id, sizeof id);
    return HPL_OK;
}

hpl_status hpl_factor(hpl_ctx *c)
{
    if (!c) return HPL_ERR_ARG;
    if (c->state != hpl_ctx::S_INIT) {
        set_err(c, "hpl_factor: context not in the initialised state");
        return HPL_ERR_STATE;
    }
    const int64_t l0 = g_launches.load();
    const int64_t nblk = cdiv(c->N, c->NB);
    if (c->timing) {
        hpl_status se = ensure_timing_events(c, nblk);
        if (se != HPL_OK) return se;
    }
    c->dgemm_flop = 0;
    c->dgemm_launches = 0;
    c->lb_base = c->lb_next;
    c->lb_next += (unsigned long long)nblk + 2;
    CK(c, cudaEventRecord(c->ev_t[0], c->s_la));
    CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_t[0], 0));
    CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_t[0], 0));
    CK(c, cudaEventRecord(c->ev_rest, c->s_tr));
    CK(c, cudaMemsetAsync(c->fw.info, 0xff, sizeof(int64_t), c->s_la));
    hpl_status s = fact_panel(c, c->s_la, 0, 0);
    if (s != HPL_OK) return s;
    CK(c, cudaEventRecord(c->ev_panel[0], c->s_la));
    // split update (option "split" = right-section percent; the paper uses 50 %,
    // PAPER.md l.66).  Default off: on B200 the RS runs as SM-driven NCCL
    // kernels over NVLink, so overlapping it with the DGEMM costs about as much
    // DGEMM throughput as it hides.
    const int split_pct = c->split_pct >= 0 ? c->split_pct : 0;
    const bool split = c->lookahead && split_pct > 0;
    int64_t split_col = c->nloc;
    if (split) {
        const int64_t n2 = std::min<int64_t>(
            c->nloc, round_up((int64_t)((double)c->nloc * split_pct / 100.0), c->NB));
        split_col = c->nloc - n2;
        CK(c, cudaEventRecord(c->ev_dgR, c->s_tr));
        CK(c, cudaEventRecord(c->ev_dgL, c->s_tr));
    }
    for (int64_t j = 0; j < nblk; ++j) {
        const int b = (int)(j % hpl_ctx::NBUF), bn = (int)((j + 1) % hpl_ctx::NBUF);
        const int64_t j0 = j * c->NB, jb = jb_of(c, j);
        const int64_t lct = lcols_before(c, j0 + jb), cend = c->nloc;  // local trailing cols
        const bool has_next = j + 1 < nblk;
        const int64_t jb1 = has_next ? jb_of(c, j + 1) : 0;
        // panel j+1 lives in the next jb1 local columns of its owner column
        const bool own_next = has_next && c->mycol == (int)((j + 1) % c->Q);
        const int64_t lrest = lct + (own_next ? jb1 : 0);
        cudaEvent_t *E = c->timing ? &c->tev[10 * j] : nullptr;
        if (c->lookahead && split) {
            // Split update: right section [cs, cend) (fixed width n2, holds b) and
            // left section [lrest, cs).  S_rs runs RS_R(j) then RS_L(j); S_tr runs
            // UPDATE_R(j) then UPDATE_L(j).  RS_L(j) overlaps UPDATE_R(j) and
            // RS_R(j+1) overlaps UPDATE_L(j).  Once the left section is used up the
            // right section is the whole rest (the paper's fallback).
            const int64_t cs = std::max(lrest, split_col);
            RsOut rsR, rsL;
            CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_panel[b], 0));
            CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_dgR, 0));
            if (E) CK(c, cudaEventRecord(E[0], c->s_rs));
            s = rs_cols(c, c->s_rs, j, b, cs, cend, SEC_RIGHT, c->col_comm_tr, &rsR);
            if (s != HPL_OK) return s;
            CK(c, cudaEventRecord(c->ev_rsR, c->s_rs));
            CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_dgL, 0));
            s = rs_cols(c, c->s_rs, j, b, lrest, cs, SEC_LEFT, c->col_comm_tr, &rsL);
            if (s != HPL_OK) return s;
            CK(c, cudaEventRecord(c->ev_rsL, c->s_rs));
            if (E) CK(c, cudaEventRecord(E[1], c->s_rs));
            CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_rsR, 0));
            s = compute_cols(c, c->s_tr, j, b, cs, cend, rsR, E ? E[2] : nullptr, E != nullptr,
                             c->ev_trsm);
            if (s != HPL_OK) return s;
            CK(c, cudaEventRecord(c->ev_dgR, c->s_tr));
            CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_rsL, 0));
            s = compute_cols(c, c->s_tr, j, b, lrest, cs, rsL, nullptr, E != nullptr);
            if (s != HPL_OK) return s;
            CK(c, cudaEventRecord(c->ev_dgL, c->s_tr));
            if (E) CK(c, cudaEventRecord(E[3], c->s_tr));
            CK(c, cudaEventRecord(c->ev_rest, c->s_tr));
            CK(c, cudaEventRecord(c->ev_next, c->s_tr));
        } else if (c->lookahead) {
            // Update panel j+2's columns (on their owner: the first rest columns)
            // before the remainder, so la(j+1) and FACT(j+2) can start while the
            // remainder of rest(j) runs: FACT(j+2) then hides behind the rest of
            // iteration j and all of iteration j+1 (SURVEY §3.4 refinement).
            CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_panel[b], 0));
            const bool has_next2 = j + 2 < nblk;
            const int64_t jb2 = has_next2 ? jb_of(c, j + 2) : 0;
            const bool own_next2 = has_next2 && c->mycol == (int)((j + 2) % c->Q);
            if (c->early_next && own_next2 && lrest + jb2 < cend) {
                s = update_cols(c, c->s_tr, j, b, lrest, lrest + jb2, nullptr, c->ev_trsm);
                if (s != HPL_OK) return s;
                CK(c, cudaEventRecord(c->ev_next, c->s_tr));
                s = update_cols(c, c->s_tr, j, b, lrest + jb2, cend, E);
                if (s != HPL_OK) return s;
            } else if (c->hp_trsm) {
                // RS + DTRSM of the rest on the high-priority S_rs (critical path),
                // only the long DGEMM at low priority on S_tr
                RsOut rs;
                CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_panel[b], 0));
                CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_rest, 0));
                if (E) CK(c, cudaEventRecord(E[0], c->s_rs));
                s = rs_cols(c, c->s_rs, j, b, lrest, cend, SEC_RIGHT, c->col_comm_tr, &rs);
                if (s != HPL_OK) return s;
                if (E) CK(c, cudaEventRecord(E[1], c->s_rs));
                // DTRSM / DGEMM pipelined over column chunks (option trsm_pipe =
                // chunk count): the DGEMM of chunk 0 starts as soon as its DTRSM is
                // done and hides the DTRSM of the remaining chunks
                const int64_t n = cend - lrest;
                int64_t w1 = n;
                if (c->trsm_pipe > 1 && n >= 8 * 1024)
                    w1 = std::min<int64_t>(n, round_up(cdiv(n, c->trsm_pipe), 64));
                s = compute_cols(c, c->s_rs, j, b, lrest, lrest + w1, rs, E ? E[2] : nullptr, false,
                                 w1 < n ? c->ev_trsm0 : c->ev_trsm, true, false);
                if (s != HPL_OK) return s;
                RsOut rs1{rs.u + w1, rs.ldu};
                if (w1 < n) {
                    s = compute_cols(c, c->s_rs, j, b, lrest + w1, cend, rs1, nullptr, false,
                                     c->ev_trsm, true, false);
                    if (s != HPL_OK) return s;
                }
                CK(c, cudaStreamWaitEvent(c->s_tr, w1 < n ? c->ev_trsm0 : c->ev_trsm, 0));
                s = compute_cols(c, c->s_tr, j, b, lrest, lrest + w1, rs, nullptr, E != nullptr,
                                 nullptr, false, true);
                if (s != HPL_OK) return s;
                if (w1 < n) {
                    CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_trsm, 0));
                    s = compute_cols(c, c->s_tr, j, b, lrest + w1, cend, rs1, nullptr, E != nullptr,
                                     nullptr, false, true);
                    if (s != HPL_OK) return s;
                }
                if (E) CK(c, cudaEventRecord(E[3], c->s_tr));
                CK(c, cudaEventRecord(c->ev_next, c->s_tr));
            } else {
                s = update_cols(c, c->s_tr, j, b, lrest, cend, E, c->ev_trsm);
                if (s != HPL_OK) return s;
                CK(c, cudaEventRecord(c->ev_next, c->s_tr));
            }
            CK(c, cudaEventRecord(c->ev_rest, c->s_tr));
        }
        if (c->lookahead) {
            if (E) CK(c, cudaEventRecord(E[4], c->s_la));
            if (own_next) {
                s = update_cols(c, c->s_la, j, b, lct, lct + jb1);
                if (s != HPL_OK) return s;
            }
            if (E) CK(c, cudaEventRecord(E[5], c->s_la));
            // FACT(j+1) competes for SMs: let the rest's LASWP + DTRSM (on the
            // critical path of S_tr) finish first; FACT then overlaps the DGEMM.
            if (has_next) CK(c, cudaStreamWaitEvent(c->s_la, c->ev_trsm, 0));
            if (has_next) {
                s = fact_panel(c, c->s_la, j + 1, bn, E ? E[7] : nullptr, E ? E[8] : nullptr);
                if (s != HPL_OK) return s;
                CK(c, cudaEventRecord(c->ev_panel[bn], c->s_la));
            }
            if (E) CK(c, cudaEventRecord(E[6], c->s_la));
            // la(j+1) touches panel j+2's columns: wait until rest(j) updated them
            CK(c, cudaStreamWaitEvent(c->s_la, c->ev_next, 0));
        } else {
            if (E) CK(c, cudaEventRecord(E[4], c->s_la));
            s = update_cols(c, c->s_la, j, b, lct, cend, E);
            if (s != HPL_OK) return s;
            if (E) CK(c, cudaEventRecord(E[5], c->s_la));
            if (has_next) {
                s = fact_panel(c, c->s_la, j + 1, bn, E ? E[7] : nullptr, E ? E[8] : nullptr);
                if (s != HPL_OK) return s;
            }
            if (E) CK(c, cudaEventRecord(E[6], c->s_la));
        }
    }
    CK(c, cudaEventRecord(c->ev_rest, c->s_tr));
    CK(c, cudaStreamWaitEvent(c->s_la, c->ev_rest, 0));
    CK(c, cudaEventRecord(c->ev_t[1], c->s_la));
    CK(c, cudaStreamSynchronize(c->s_la));
    CK(c, cudaStreamSynchronize(c->s_tr));
    c->launches = g_launches.load() - l0;
    c->factor_ms = ev_ms(c->ev_t[0], c->ev_t[1]);
    c->timeline.clear();
    c->fact_detail.clear();
    c->dgemm_ms = 0;
    if (c->timing) {
        c->timeline.reserve(6 * nblk);
        c->fact_detail.reserve(3 * nblk);
        for (int64_t j = 0; j < nblk; ++j) {
            cudaEvent_t *E = &c->tev[10 * j];
            const double rest_dg = ev_ms(E[2], E[3]);
            c->timeline.push_back(c->lookahead ? ev_ms(E[5], E[6]) : ev_ms(E[5], E[6]));
            c->timeline.push_back(ev_ms(E[4], E[5]));
            c->timeline.push_back(ev_ms(E[0], E[3]));
            c->timeline.push_back(ev_ms(E[0], E[1]));
            c->timeline.push_back(ev_ms(E[1], E[2]));
            c->timeline.push_back(rest_dg);
            c->dgemm_ms += rest_dg;
            const bool nx = j + 1 < nblk;
            c->fact_detail.push_back(nx ? ev_ms(E[5], E[7]) : 0.0);
            c->fact_detail.push_back(nx ? ev_ms(E[7], E[8]) : 0.0);
            c->fact_detail.push_back(nx ? ev_ms(E[8], E[6]) : 0.0);
        }
    }
    if (c->dist) {
        // the owner column saw the zero pivot: min over all ranks (unsigned: -1 = none)
        NK(c, ncclAllReduce(c->fw.info, c->fw.info, 1, ncclUint64, ncclMin, c->world, c->s_la));
        CK(c, cudaStreamSynchronize(c->s_la));
    }
    int64_t info = -1;
    CK(c, cudaMemcpy(&info, c->fw.info, sizeof info, cudaMemcpyDeviceToHost));
    c->state = hpl_ctx::S_FACTORED;
    if (info != -1) {
        c->singular = info;
        set_err(c, "exact zero pivot in global column %lld", (long long)info);
        return HPL_ERR_SINGULAR;
    }
    return HPL_OK;
}

hpl_status hpl_solve(hpl_ctx *c, double *x_host)
{
    if (!c) return HPL_ERR_ARG;
    if (c->state != hpl_ctx::S_FACTORED) {
        set_err(c, "hpl_solve: call hpl_factor first");
        return HPL_ERR_STATE;
    }
    if (c->singular >= 0) return HPL_ERR_SINGULAR;
    const int64_t l0 = g_launches.load();
    CK(c, cudaEventRecord(c->ev_t[1], c->s_la));
    {
        // Distributed block back substitution.  Block row bb lives on process
        // row rb = bb mod P: its Q processes form the partial sums over their
        // local columns (all-reduce on the row comm), the owner of the
        // diagonal block (rb, bb mod Q) solves it, and x_b is broadcast to
        // every rank (world comm) so x stays replicated.
        const int64_t N = c->N, nblk = cdiv(N, c->NB);
        const int ycol = (int)((N / c->NB) % c->Q);            // owner of global column N
        const int64_t lcy = c->mycol == ycol ? lcols_before(c, N) : -1;
        const int64_t lcN = lcols_before(c, N);
        for (int64_t bb = nblk - 1; bb >= 0; --bb) {
            const int64_t r0 = bb * c->NB, r1 = std::min<int64_t>(N, r0 + c->NB);
            const int nb = (int)(r1 - r0);
            const int rb = (int)(bb % c->P), qb = (int)(bb % c->Q);
            if (c->myrow == rb) {
                const int64_t lr0 = lrows_before(c, r0);
                // every rank of the process row uses the same split count
                // (a function of the global sizes) so the all-reduce lines up
                const int S = bs_splits(nb, 0, cdiv(cdiv(N - r1, c->NB), c->Q) * c->NB, c->NB);
                CK(c, bs_partial(c->s_la, nb, c->A + lr0 * c->lda, c->lda,
                                       lcols_before(c, r1), lcN, c->NB, c->Q, c->mycol, c->x,
                                       lcy, c->tbuf, S));
                if (c->Q > 1)
                    NK(c, ncclAllReduce(c->tbuf, c->tbuf, (size_t)S * nb, ncclDouble, ncclSum,
                                        c->row_comm, c->s_la));
                if (c->mycol == qb)
                    CK(c, bs_diag(c->s_la, nb, c->A + lr0 * c->lda + lcols_before(c, r0), c->lda,
                                  c->tbuf, S, c->x + r0));
            }
            if (c->dist)
                NK(c, ncclBroadcast(c->x + r0, c->x + r0, nb, ncclDouble, rb + qb * c->P,
                                    c->world, c->s_la));
        }
    }
    if (x_host)
        CK(c, cudaMemcpyAsync(x_host, c->x, sizeof(double) * c->N, cudaMemcpyDeviceToHost,
                              c->s_la));
    CK(c, cudaEventRecord(c->ev_t[2], c->s_la));
    CK(c, cudaStreamSynchronize(c->s_la));
    c->solve_ms = ev_ms(c->ev_t[1], c->ev_t[2]);
    c->launches += g_launches.load() - l0;
    c->state = hpl_ctx::S_SOLVED;
    return HPL_OK;
}

hpl_status hpl_residual(hpl_ctx *c, double *resid)
{
    if (!c || !resid) return HPL_ERR_ARG;
    if (c->state != hpl_ctx::S_SOLVED) {
        set_err(c, "hpl_residual: call hpl_solve first");
        return HPL_ERR_STATE;
    }
    // r and the row sums of |A0| for this process row's rows, summed over the
    // process row; the norms are then maxed over the process column.
    CK(c, residual_partial(c->s_la, c->seed, c->N, c->NB, c->P, c->myrow, c->mloc, c->Q,
                           c->mycol, lcols_before(c, c->N), c->x, c->rvec, c->avec));
    if (c->Q > 1) {
        NK(c, ncclAllReduce(c->rvec, c->rvec, c->mloc, ncclDouble, ncclSum, c->row_comm, c->s_la));
        NK(c, ncclAllReduce(c->avec, c->avec, c->mloc, ncclDouble, ncclSum, c->row_comm, c->s_la));
    }
    CK(c, residual_finalize(c->s_la, c->seed, c->N, c->NB, c->P, c->myrow, c->mloc, c->rvec,
                            c->avec, c->x, c->out4));
    if (c->dist)
        NK(c, ncclAllReduce(c->out4, c->out4, 4, ncclDouble, ncclMax, c->world, c->s_la));
    double h[4];
    CK(c, cudaMemcpyAsync(h, c->out4, sizeof h, cudaMemcpyDeviceToHost, c->s_la));
    CK(c, cudaStreamSynchronize(c->s_la));
    const double eps = 0x1p-53;
    *resid = h[0] / (eps * (h[1] * h[2] + h[3]) * (double)c->N);
    return HPL_OK;
}

hpl_status hpl_regenerate(hpl_ctx *c)
{
    if (!c || !c->A) return HPL_ERR_ARG;
    c->singular = -1;
    return generate(c);
}

hpl_status hpl_load_local(hpl_ctx *c, const double *host, int64_t ld)
{
    if (!c || !host || ld < c->nloc) return HPL_ERR_ARG;
    CK(c, cudaMemcpy2DAsync(c->A, c->lda * 8, host, ld * 8, c->nloc * 8, c->mloc,
                            cudaMemcpyHostToDevice, c->s_tr));
    CK(c, cudaStreamSynchronize(c->s_tr));
    c->singular = -1;
    c->state = hpl_ctx::S_INIT;
    return HPL_OK;
}

hpl_status hpl_local_shape(const hpl_ctx *c, int64_t *rows, int64_t *cols)
{
    if (!c) return HPL_ERR_ARG;
    if (rows) *rows = c->mloc;
    if (cols) *cols = c->nloc;
    return HPL_OK;
}

void hpl_free(hpl_ctx *c)
{
    if (!c) return;
    if (c->s_la) cudaStreamSynchronize(c->s_la);
    if (c->s_tr) cudaStreamSynchronize(c->s_tr);
    release(c);
    delete c;
}

const char *hpl_last_error(const hpl_ctx *c) { return c ? c->err.c_str() : "null context"; }

int64_t hpl_singular_column(const hpl_ctx *c) { return c ? c->singular : -1; }

hpl_status hpl_get_ipiv(const hpl_ctx *c, int64_t *ipiv_host)
{
    if (!c || !ipiv_host) return HPL_ERR_ARG;
    if (c->state < hpl_ctx::S_FACTORED) return HPL_ERR_STATE;
    if (cudaMemcpy(ipiv_host, c->gpiv, sizeof(int64_t) * c->N, cudaMemcpyDeviceToHost) !=
        cudaSuccess)
        return HPL_ERR_CUDA;
    return HPL_OK;
}

hpl_status hpl_get_local(const hpl_ctx *c, double *host, int64_t ld)
{
    if (!c || !host || ld < c->nloc) return HPL_ERR_ARG;
    if (cudaMemcpy2D(host, ld * 8, c->A, c->lda * 8, c->nloc * 8, c->mloc,
                     cudaMemcpyDeviceToHost) != cudaSuccess)
        return HPL_ERR_CUDA;
    return HPL_OK;
}

int64_t hpl_get_timeline(const hpl_ctx *c, double *t, int64_t cap)
{
    if (!c || !t) return 0;
    const int64_t n = std::min<int64_t>(cap, (int64_t)c->timeline.size() / 6);
    std::memcpy(t, c->timeline.data(), sizeof(double) * 6 * n);
    return n;
}

int64_t hpl_get_fact_detail(const hpl_ctx *c, double *t, int64_t cap)
{
    if (!c || !t) return 0;
    const int64_t n = std::min<int64_t>(cap, (int64_t)c->fact_detail.size() / 3);
    std::memcpy(t, c->fact_detail.data(), sizeof(double) * 3 * n);
    return n;
}

hpl_status hpl_set_timing(hpl_ctx *c, int32_t enable)
{
    if (!c) return HPL_ERR_ARG;
    c->timing = enable != 0;
    return HPL_OK;
}

hpl_status hpl_set_option(hpl_ctx *c, const char *name, int64_t value)
{
    if (!c || !name) return HPL_ERR_ARG;
    if (!strcmp(name, "lookahead")) c->lookahead = value != 0;
    else if (!strcmp(name, "nbmin")) {
        if (value < 1 || value > 16) return HPL_ERR_ARG;
        c->nbmin = (int)value;
    } else if (!strcmp(name, "gemm_cfg")) dgemm_set_default_cfg((int)value);
    else if (!strcmp(name, "gemm_tpc")) dgemm_set_tiles_per_cta((int)value);
    else if (!strcmp(name, "gemm_red")) dgemm_set_red_epilogue((int)value);
    else if (!strcmp(name, "leaf_ctas")) {
        c->leaf_auto = false;
        fact_set_leaf_warp_ctas(0);
        fact_set_leaf_ctas((int)value, 0);
    } else if (!strcmp(name, "leaf_warp")) { c->leaf_auto = true; c->leaf_warp = (int)value; }
    else if (!strcmp(name, "leaf_rows")) { c->leaf_auto = false; fact_set_leaf_ctas(-1, (int)value); }
    else if (!strcmp(name, "split")) c->split_pct = (int)value;
    else if (!strcmp(name, "early_next")) c->early_next = value != 0;
    else if (!strcmp(name, "hp_trsm")) c->hp_trsm = value != 0;
    else if (!strcmp(name, "rs_peer")) c->rs_peer = value != 0 && c->rsflag != nullptr;
    else if (!strcmp(name, "store_l")) c->store_l = value != 0;
    else if (!strcmp(name, "la_below_rs")) {     // between factorizations only
        cudaStreamSynchronize(c->s_la);
        c->s_la = value ? c->s_la_mid : c->s_la_hi;
    }
    else if (!strcmp(name, "leaf_cluster")) fact_set_leaf_cluster((int)value);   // process-wide
    else if (!strcmp(name, "fact_gather")) c->fact_gather_rows = std::max<int64_t>(0, value);
    else if (!strcmp(name, "fact_gather_ms")) c->fact_gather_ms = (double)value;
    else if (!strcmp(name, "leaf_variant")) {   // process-wide (like the gemm_* knobs)
        if (value < 0 || value > 2) return HPL_ERR_ARG;
        fact_set_leaf_variant((int)value);
    }
    else if (!strcmp(name, "trsm_pipe")) c->trsm_pipe = (int)std::max<int64_t>(1, value);
    else if (!strcmp(name, "lb_peer")) c->lb_peer = value != 0 && c->lbflag != nullptr;
    else if (!strcmp(name, "leaf_few_ctas")) { c->leaf_auto = true; c->leaf_few_ctas = (int)value; }
    else if (!strcmp(name, "leaf_hide_ms")) { c->leaf_auto = true; c->leaf_hide_ms = (double)value; }
    else return HPL_ERR_ARG;
    return HPL_OK;
}

int64_t hpl_launch_count(const hpl_ctx *c) { return c ? c->launches : 0; }

hpl_status hpl_plan_fact(int64_t N, int32_t NB, int32_t P, int32_t Q, int32_t myrow, int64_t j,
                         int64_t gather_rows, double gather_ms, int64_t *out5)
{
    if (!out5 || N < 1 || NB < 1 || P < 1 || Q < 1 || myrow < 0 || myrow >= P || j < 0 ||
        j * NB >= N)
        return HPL_ERR_ARG;
    int64_t lrL0, mL, ldp;
    fact_geom(N, NB, P, myrow, j, &lrL0, &mL, &ldp);
    out5[0] = P < 2 ? -1
                    : use_gathered_fact(N, NB, P, Q, j, gather_rows, gather_ms,
                                        std::min<int64_t>(N, (int64_t)1 << 16)) ? 1 : 0;
    out5[1] = N - j * NB;                   // global rows of the panel (T + all L rows)
    out5[2] = lrL0;                         // this process row's first L row (local)
    out5[3] = mL;                           // this process row's L rows
    out5[4] = ldp;                          // leading dimension of its packed panel
    return HPL_OK;
}

hpl_status hpl_plan_iteration(int64_t N, int32_t NB, int32_t P, int32_t Q, int32_t myrow,
                              int32_t mycol, int64_t j, int64_t *out8)
{
    if (!out8 || N < 1 || NB < 1 || P < 1 || Q < 1 || myrow < 0 || myrow >= P || mycol < 0 ||
        mycol >= Q || j < 0 || j * NB >= N)
        return HPL_ERR_ARG;
    hpl_ctx t;
    t.N = N; t.NB = NB; t.P = P; t.Q = Q; t.myrow = myrow; t.mycol = mycol;
    t.mloc = numroc(N, NB, myrow, P);
    t.nloc = numroc(N + 1, NB, mycol, Q);
    const int64_t nblk = cdiv(N, NB);
    const int64_t j0 = j * NB, jb = jb_of(&t, j);
    const int64_t lct = lcols_before(&t, j0 + jb);
    const bool has_next = j + 1 < nblk;
    const int64_t jb1 = has_next ? jb_of(&t, j + 1) : 0;
    const bool own_next = has_next && mycol == (int)((j + 1) % Q);
    out8[0] = lrows_before(&t, j0);            // first active local row
    out8[1] = lct;                             // first trailing local column
    out8[2] = own_next ? lct : lct;            // look-ahead range begin
    out8[3] = own_next ? lct + jb1 : lct;      // look-ahead range end
    out8[4] = lct + (own_next ? jb1 : 0);      // rest range begin
    out8[5] = t.nloc;                          // rest range end
    out8[6] = (int)(j % Q) == mycol ? lcols_before(&t, j0) : -1;  // local panel column (owner)
    out8[7] = jb;
    return HPL_OK;
}

hpl_status hpl_pin_host(void *p, int64_t bytes, int32_t pin)
{
    if (!p || bytes <= 0) return HPL_ERR_ARG;
    cudaError_t e = pin ? cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault)
                        : cudaHostUnregister(p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return HPL_ERR_CUDA;
    }
    return HPL_OK;
}

hpl_status hpl_last_timing(const hpl_ctx *c, double *out6)
{
    if (!c || !out6) return HPL_ERR_ARG;
    out6[0] = c->factor_ms;
    out6[1] = c->solve_ms;
    out6[2] = (double)c->dgemm_launches;
    out6[3] = c->dgemm_ms;
    out6[4] = c->dgemm_flop;
    out6[5] = (double)c->launches;
    return HPL_OK;
}

}  // extern "C"
