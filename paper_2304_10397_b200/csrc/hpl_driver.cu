// hpl_driver.cu — the per-iteration schedule and the rest of the C ABI
// (include/hpl.h).  Process grid, peer memory and collectives: hpl_comm.cu.
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
// columns and FACT(j+1) run on a high-priority stream S_la; the RS + DTRSM of
// the remaining columns on a second high-priority stream S_rs and their
// DGEMM on the low-priority S_tr; events order them.  The
// split update is the one alternative schedule: S_rs runs
// the RS of the right section, then of the left one, while S_tr updates them.
//
// Distribution: 2D block-cyclic over P x Q (rank = p + q*P).
// FACT runs on the process column that owns panel j (P > 1: pivot exchange
// inside the leaf over peer memory, or the gathered FACT for small panels);
// the packed panel (with its pivots) reaches the process row by a copy-engine
// pull over peer memory (LBCAST: "Processes which do not
// participate in the FACT phase simply wait in the LBCAST phase"); the row
// swaps cross process rows as a peer-memory gather (RS).
#include "hpl_ctx.cuh"
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <ctime>

using namespace hpl;

namespace {

// HPL_TRACE=1: host-side timestamps of the collective calls, recorded in the
// context (no I/O on the way) and printed by hpl_free — for diagnosing
// loopback stalls; off by default.
void trace(hpl_ctx *c, const char *what, long long k = -1)
{
    static const bool on = getenv("HPL_TRACE") != nullptr;
    if (!on || c->trace_n >= (int)(sizeof c->trace_t / sizeof c->trace_t[0])) return;
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    c->trace_t[c->trace_n] = ts.tv_sec * 1000000000ll + ts.tv_nsec;
    c->trace_w[c->trace_n] = what;
    c->trace_k[c->trace_n++] = k;
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
        CK(c, cm_to_rm(st, jb + mL, jb, c->panel[b], ldpj, Ablk, c->lda));
        return HPL_OK;
    }
    // T from the owner of block row j to the whole process column
    if (is_prow) CK(c, rm_to_cm(st, jb, jb, c->A + lr0 * c->lda + lcp, c->lda, c->Tbuf, jb));
    ST(coll_bcast(c, G_COL, c->Tbuf, sizeof(double) * (size_t)(jb * jb), prow_of(c, j), st));
    ST(d2d_2d(c, st, c->panel[b], ldpj * 8, c->Tbuf, jb * 8, jb * 8, jb));
    CK(c, rm_to_cm(st, mL, jb, c->A + lrL0 * c->lda + lcp, c->lda, c->panel[b] + jb, ldpj));
    const int64_t rows_total = c->N - j0;   // T + every process row's L rows
    if (use_gathered_fact(c->N, c->NB, c->P, c->Q, j, c->fact_gather_rows, c->fact_gather_ms,
                          c->cp_max_rows)) {
        // Gathered FACT: barrier (every packed panel of the column is ready),
        // build the combined panel from peer memory, barrier (every peer has
        // read this panel), factor it here (the same arithmetic the
        // distributed leaf performs, so the same bits), keep this process's rows.
        const unsigned long long v = ++c->fg_seq;
        CK(c, rs_barrier(st, c->rsp, 6, v, spin(c)));
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
        CK(c, rs_barrier(st, c->rsp, 7, v, spin(c)));
        if (c->leaf_auto) {
            fact_set_leaf_ctas(&c->fw, 0, 512);       // on the critical path: every SM
            c->fw.leaf_warp_ctas = c->loop ? c->fw.max_ctas : 0;
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
        CK(c, panel_fact(st, jb + mL, jb, c->panel[b], ldpj, panel_ipiv(c, j, b), c->nbmin,
                         &c->fw, c->scratch, j0, &df));
    }
    CK(c, cm_to_rm(st, mL, jb, c->panel[b] + jb, ldpj, c->A + lrL0 * c->lda + lcp, c->lda));
    if (is_prow) CK(c, cm_to_rm(st, jb, jb, c->panel[b], ldpj, c->A + lr0 * c->lda + lcp, c->lda));
    return HPL_OK;
}

// Panel j is about to be written into this rank's panel[j % nbuf] (by FACT on
// the owner, by the LBCAST copy elsewhere).  If this rank owned panel
// j - nbuf, the other columns may still be pulling it from that buffer: wait
// until every one of them has copied it (their done words in this rank's
// lbflag).  Owners of j - nbuf are the only ranks whose buffer peers read.
hpl_status wait_panel_buffer_free(hpl_ctx *c, cudaStream_t st, int64_t j)
{
    if (c->Q == 1 || !c->lb_peer || j < c->nbuf) return HPL_OK;
    const int64_t jo = j - c->nbuf;
    if ((int)(jo % c->Q) != c->mycol) return HPL_OK;
    FlagOp op{};
    for (int q = 0; q < c->Q; ++q)
        if (q != c->mycol) op.wt[op.nwait++] = c->lbflag + hpl_ctx::LB_DONE + q;
    op.wv = c->lb_base + (unsigned long long)jo + 1;
    CK(c, flag_op(st, op, spin(c)));
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
            CK(c, flag_op(st, op, spin(c)));
        } else {
            ST(wait_panel_buffer_free(c, st, j));
            op.wt[op.nwait++] = c->lbflag + pcol;
            op.wv = c->lb_base + (unsigned long long)j + 1;
            CK(c, flag_op(st, op, spin(c)));
            ST(d2d(c, st, c->panel[b], c->ppanel[pcol * hpl_ctx::MAXBUF + b], pbytes));
            FlagOp done{};
            done.sig[done.nsig++] = c->pflag[pcol] + hpl_ctx::LB_DONE + c->mycol;
            done.sv = c->lb_base + (unsigned long long)j + 1;
            CK(c, flag_op(st, done, spin(c)));
        }
    } else if (c->Q > 1) {
        ST(coll_bcast(c, G_ROW, c->panel[b], pbytes, pcol, st));
    }
    // the plan is in GLOBAL rows (P = 1: global == local)
    CK(c, pivot_plan(st, jb, j0, panel_ipiv(c, j, b), j0, c->N, c->gpiv + j0, c->src[b],
                     c->disp[b], c->ndisp[b]));
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
        // FACT(0) has nothing to hide behind: it always gets every SM; nor
        // has any FACT without look-ahead (the update before it is done)
        const bool hide = c->lookahead && j > 0 && rest_ms > c->leaf_hide_ms;
        fact_set_leaf_ctas(&c->fw, hide ? c->leaf_few_ctas : 0, 512);
        c->fw.leaf_warp_ctas = hide ? c->leaf_warp : 0;
        // loopback: one-warp leaf CTAs only.  A 256-thread leaf CTA needs a
        // whole SM's registers and starved behind the other ranks' DGEMM CTAs
        // while its peers spun (P >= 4: 10-25 % of runs timed out); a one-warp
        // CTA fits beside three DGEMM CTAs (bitwise-equal results, tested)
        if (c->loop) c->fw.leaf_warp_ctas = c->fw.max_ctas;
    }
    if (c->mycol == (int)(j % c->Q)) {
        ST(wait_panel_buffer_free(c, st, j));
        ST(fact_local(c, st, j, b));
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
// final block rows, each from its owner; W = the original block row from its
// owner, for the displaced rows).
hpl_status rs_cols(hpl_ctx *c, cudaStream_t st, int64_t j, int b, int64_t c0, int64_t c1, int sec,
                   RsOut *out)
{
    const int64_t j0 = j * c->NB, jb = jb_of(c, j), n = c1 - c0;
    out->u = c->U + ucol(c0);
    out->ldu = c->ldu;
    if (n <= 0) return HPL_OK;
    if (c->P == 1) {
        CK(c, laswp_gather_scatter(st, jb, c->src[b], c->disp[b], c->ndisp[b], c->A, c->lda, c0,
                                   c1, out->u, c->ldu));
        return HPL_OK;
    }
    const int64_t lr0 = lrows_before(c, j0);
    const int64_t ldub = round_up(n, 16);
    double *u = c->Ub[sec], *w = c->Wb[sec];
    out->u = u;
    out->ldu = ldub;
    if (c->rs_peer) {
        // peer memory: barrier (peers' columns are at iteration j), gather U and
        // this process's W rows over NVLink, barrier (peers done reading), scatter
        const unsigned long long v = ++c->rs_seq[sec];
        CK(c, rs_barrier(st, c->rsp, 2 * sec, v, spin(c)));
        CK(c, rs_gather_peer(st, jb, c->src[b], c->disp[b], c->ndisp[b], c->rsp, c->lda, c0, c1,
                             u, ldub, w, ldub, j0, c->NB));
        CK(c, rs_barrier(st, c->rsp, 2 * sec + 1, v, spin(c)));
        CK(c, rs_scatter(st, c->disp[b], c->ndisp[b], w, ldub, j0, c->A, c->lda, c0, c1, c->NB,
                         c->P, c->myrow));
        return HPL_OK;
    }
    // collective variant: U summed over the process column (zeros where a
    // process does not own the row), W broadcast from the owner of block row j
    const int gid = sec == SEC_LA ? G_COL : G_COLTR;
    CK(c, rs_pack(st, jb, c->src[b], c->A, c->lda, c0, c1, u, ldub, c->NB, c->P, c->myrow));
    if (c->myrow == prow_of(c, j))
        ST(d2d_2d(c, st, w, ldub * 8, c->A + lr0 * c->lda + c0, c->lda * 8, n * 8, jb));
    ST(coll_allreduce(c, gid, u, jb * ldub, COLL_SUM, st));
    ST(coll_bcast(c, gid, w, sizeof(double) * (size_t)(jb * ldub), prow_of(c, j), st));
    CK(c, rs_scatter(st, c->disp[b], c->ndisp[b], w, ldub, j0, c->A, c->lda, c0, c1, c->NB, c->P,
                     c->myrow));
    return HPL_OK;
}

int slot_of(const hpl_ctx *c, cudaStream_t st)
{
    return st == c->s_la ? SLOT_LOOKAHEAD : st == c->s_rs ? SLOT_RS : SLOT_TRAIL;
}

// DTRSM (do_trsm) and/or DGEMM (do_gemm) of iteration j for local columns
// [c0, c1) once RS(j) has produced U.
hpl_status compute_cols(hpl_ctx *c, cudaStream_t st, int64_t j, int b, int64_t c0, int64_t c1,
                        const RsOut &rs, bool do_trsm, bool do_gemm, bool count)
{
    const int64_t n = c1 - c0;
    if (n <= 0) return HPL_OK;
    const int slot = slot_of(c, st);
    const int64_t j0 = j * c->NB, jb = jb_of(c, j);
    const int64_t lr0 = lrows_before(c, j0), lrL0 = lrL0_of(c, j), ldpj = panel_ld(c, j);
    double *u2 = c->U2 + ucol(c0);
    // block row j <- L11^{-1} U: into U2 (the DGEMM operand) and, on the owner
    // of block row j, into A as well
    if (do_trsm) {
        if (c->myrow == prow_of(c, j))
            CK(c, dgemm(st, GEMM_ASSIGN, true, jb, n, jb, c->linv[b], c->ldlinv, rs.u, rs.ldu,
                        c->A + lr0 * c->lda + c0, c->lda, c->gemm_cfg, u2, c->ldu, slot));
        else
            CK(c, dgemm(st, GEMM_ASSIGN, true, jb, n, jb, c->linv[b], c->ldlinv, rs.u, rs.ldu, u2,
                        c->ldu, c->gemm_cfg, nullptr, 0, slot));
        if (count) c->trsm_flop += (double)jb * (double)jb * (double)n;
    }
    const int64_t mrest = c->mloc - lrL0;
    if (mrest > 0 && do_gemm) {
        CK(c, dgemm(st, GEMM_UPDATE, false, mrest, n, jb, c->panel[b] + jb, ldpj, u2, c->ldu,
                    c->A + lrL0 * c->lda + c0, c->lda, c->gemm_cfg, nullptr, 0, slot));
        if (count) {
            c->dgemm_flop += 2.0 * (double)mrest * (double)n * (double)jb;
            c->dgemm_launches += 1;
        }
    }
    return HPL_OK;
}

// UPDATE(j) of local columns [c0, c1) on one stream: RS, DTRSM, DGEMM.
hpl_status update_cols(hpl_ctx *c, cudaStream_t st, int64_t j, int b, int64_t c0, int64_t c1,
                       int sec)
{
    RsOut rs;
    ST(rs_cols(c, st, j, b, c0, c1, sec, &rs));
    return compute_cols(c, st, j, b, c0, c1, rs, true, true, false);
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

bool usable(hpl_ctx *c, int want, const char *who)
{
    if (c->state == hpl_ctx::S_BROKEN) {
        set_err(c, "%s: the context is broken by an earlier peer timeout; free it", who);
        return false;
    }
    return c->state == want;
}

// The local [A | b] arriving from a host buffer (hpl_load_factor).
struct Arrival {
    const double *host;
    int64_t ld;
};

// Pipelined start (hpl_load_factor): the local matrix is copied in column
// chunks (whole NB blocks) on a copy stream while the first K iterations run
// chunk by chunk on S_la.  The first K+1 chunks are one local block each, so
// FACT(0) starts after one block has landed and FACT(j) follows as soon as
// the block holding panel j has received updates 0..j-1; the later chunks,
// growing from 2 to 16 blocks, receive their K updates each as they land.  Per
// column the same kernels run in the same order as in the look-ahead loop,
// so the result is bitwise that of hpl_load_local + hpl_factor (tested); the
// copy of the later chunks hides behind the earlier chunks' updates.  (A
// first version ran every chunk on its own stream: the FACT chain's kernels,
// which need whole SMs, starved behind the stream of DGEMM CTAs; a second
// one used 16 equal chunks, chunk 0 holding panels 0..K: 8.6 GB landed
// before FACT(0) could start — DESIGN.md §5.)  On return FACT(K) is done.
// Several ranks: every rank runs FACT/LBCAST(0..K) in order; the updates a
// rank applies depend only on its process column (same nloc, hence the same
// chunks), so the RS barriers pair up within a process column; a rank
// signals an RS barrier only after its own chunk has landed, so the peer rows
// it gathers are in place.  K and nbuf are the same on every rank.
hpl_status pipelined_start(hpl_ctx *c, const Arrival &a, int64_t *jstart)
{
    const int64_t nblk = cdiv(c->N, c->NB);
    const int K = (int)std::min<int64_t>(std::min<int64_t>(6, c->nbuf - 1), nblk - 1);
    const int64_t nbl_cols = cdiv(c->nloc, c->NB);            // local column blocks (b included)
    // chunks: K+1 single blocks, then 2, 3, 4, ... blocks up to 16.  A block's
    // K updates take ~1.2x its copy (C2: 11.7 vs 10 ms), so chunks that grow
    // by less than that keep the next chunk landing before the GPU needs it
    // (equal ~16-block chunks left the GPU idle ~120 ms waiting for the first)
    std::vector<int64_t> cb;
    const int64_t lead = std::min<int64_t>(K + 1, nbl_cols);
    for (int64_t x = 0; x < lead; ++x) cb.push_back(x * c->NB);
    for (int64_t x = lead, sz = 2; x < nbl_cols; x += sz, sz = std::min<int64_t>(16, sz + 1))
        cb.push_back(x * c->NB);
    cb.push_back(c->nloc);
    const int nc = (int)cb.size() - 1;
    int lo_p, hi_p;
    CK(c, cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
    if (!c->s_h2d) CK(c, cudaStreamCreateWithPriority(&c->s_h2d, cudaStreamNonBlocking, lo_p));
    while ((int)c->ev_arr.size() < nc) {
        cudaEvent_t e;
        CK(c, cudaEventCreate(&e));                  // timed: hpl_phase_stats h2d_ms
        c->ev_arr.push_back(e);
    }
    CK(c, cudaStreamWaitEvent(c->s_h2d, c->ev_t[0], 0));
    for (int k = 0; k < nc; ++k) {
        CK(c, cudaMemcpy2DAsync(c->A + cb[k], c->lda * 8, a.host + cb[k], a.ld * 8,
                                (cb[k + 1] - cb[k]) * 8, c->mloc, cudaMemcpyHostToDevice,
                                c->s_h2d));
        CK(c, cudaEventRecord(c->ev_arr[k], c->s_h2d));
    }
    cudaStream_t st = c->s_la;
    const bool auto0 = c->leaf_auto;
    const int lmax0 = c->fw.leaf_max_ctas, lrows0 = c->fw.leaf_rows_per_cta, lwarp0 = c->fw.leaf_warp_ctas;
    std::vector<int> applied(nc, 0);        // chunk k has received updates 0..applied[k]-1
    int arrived = 0;                        // S_la waits for chunks [0, arrived)
    auto arrive = [&](int k) -> hpl_status {
        for (; arrived <= k; ++arrived) CK(c, cudaStreamWaitEvent(st, c->ev_arr[arrived], 0));
        return HPL_OK;
    };
    auto update = [&](int64_t j, int k) -> hpl_status {
        const int b = (int)(j % c->nbuf);
        const int64_t lo = std::max(lcols_before(c, j * c->NB + jb_of(c, j)), cb[k]);
        const int64_t hi = cb[k + 1];
        if (lo >= hi) return HPL_OK;
        RsOut rs;
        ST(rs_cols(c, st, j, b, lo, hi, SEC_RIGHT, &rs));
        return compute_cols(c, st, j, b, lo, hi, rs, true, true, c->timing);
    };
    // bring chunk k up to date through update upto-1
    auto catch_up = [&](int k, int upto) -> hpl_status {
        ST(arrive(k));
        for (; applied[k] < upto; ++applied[k]) ST(update(applied[k], k));
        return HPL_OK;
    };
    // FACT(0..K) — alone on the GPU, so the leaf gets every SM
    c->leaf_auto = false;
    fact_set_leaf_ctas(&c->fw, 0, 512);
    c->fw.leaf_warp_ctas = c->loop ? c->fw.max_ctas : 0;   // loopback: fact_panel
    for (int64_t j = 0; j <= K; ++j) {
        if (c->mycol == (int)(j % c->Q)) {
            // the chunk holding panel j's local columns, updated by 0..j-1
            const int64_t lc = lcols_before(c, j * c->NB);
            int k = 0;
            while (cb[k + 1] <= lc) ++k;
            ST(catch_up(k, (int)j));
        }
        ST(fact_panel(c, st, j, (int)(j % c->nbuf)));
    }
    c->leaf_auto = auto0;
    c->fw.leaf_max_ctas = lmax0;
    c->fw.leaf_rows_per_cta = lrows0;
    c->fw.leaf_warp_ctas = lwarp0;
    CK(c, cudaEventRecord(c->ev_panel[K % c->nbuf], st));
    // every chunk: the rest of updates 0..K-1, in arrival order
    for (int k = 0; k < nc; ++k) ST(catch_up(k, K));
    c->h2d_bytes = 8.0 * (double)c->mloc * (double)c->nloc;
    c->h2d_last = nc - 1;
    // the look-ahead loop continues from iteration K on the whole matrix
    CK(c, cudaEventRecord(c->ev_rest, st));
    CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_rest, 0));
    CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_rest, 0));
    CK(c, cudaEventRecord(c->ev_rest, c->s_tr));
    CK(c, cudaEventRecord(c->ev_t[2], st));          // end of the pipelined start (stats)
    c->pstart_k = K;
    *jstart = K;
    return HPL_OK;
}

hpl_status factor_impl(hpl_ctx *c, const Arrival *arr)
{
    CK(c, cudaSetDevice(c->device));
    trace(c, "factor start");
    const int64_t l0 = t_launches;
    const int64_t nblk = cdiv(c->N, c->NB);
    if (c->timing) ST(ensure_timing_events(c, nblk));
    c->dgemm_flop = c->trsm_flop = 0;
    c->dgemm_launches = 0;
    c->lb_base = c->lb_next;
    c->lb_next += (unsigned long long)nblk + 2;
    CK(c, cudaEventRecord(c->ev_t[0], c->s_la));
    CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_t[0], 0));
    CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_t[0], 0));
    CK(c, cudaEventRecord(c->ev_rest, c->s_tr));
    CK(c, fill_u64(c->s_la, reinterpret_cast<unsigned long long *>(c->fw.info), ~0ull));
    int64_t jstart = 0;
    c->h2d_last = -1;
    if (arr) {
        ST(pipelined_start(c, *arr, &jstart));
    } else {
        ST(fact_panel(c, c->s_la, 0, 0));
        CK(c, cudaEventRecord(c->ev_panel[0], c->s_la));
    }
    // split update (option "split" = right-section percent; the paper uses 50 %,
    // PAPER.md l.66).  Default off: measured neutral on B200.
    const bool split = c->lookahead && c->split_pct > 0;
    int64_t split_col = c->nloc;
    if (split) {
        const int64_t n2 = std::min<int64_t>(
            c->nloc, round_up((int64_t)((double)c->nloc * c->split_pct / 100.0), c->NB));
        split_col = c->nloc - n2;
        CK(c, cudaEventRecord(c->ev_dgR, c->s_tr));
        CK(c, cudaEventRecord(c->ev_dgL, c->s_tr));
    }
    int *nd_hist = nullptr;       // displaced rows per panel (LASWP bytes), timing only
    if (c->timing) CK(c, cudaMallocAsync((void **)&nd_hist, sizeof(int) * nblk, c->s_la));
    for (int64_t j = jstart; j < nblk; ++j) {
        const int b = (int)(j % c->nbuf), bn = (int)((j + 1) % c->nbuf);
        const int64_t j0 = j * c->NB, jb = jb_of(c, j);
        const int64_t lct = lcols_before(c, j0 + jb), cend = c->nloc;  // local trailing cols
        const bool has_next = j + 1 < nblk;
        const int64_t jb1 = has_next ? jb_of(c, j + 1) : 0;
        // panel j+1 lives in the next jb1 local columns of its owner column
        const bool own_next = has_next && c->mycol == (int)((j + 1) % c->Q);
        const int64_t lrest = lct + (own_next ? jb1 : 0);
        cudaEvent_t *E = c->timing ? &c->tev[10 * j] : nullptr;
        if (E) ST(d2d(c, c->s_la, nd_hist + j, c->ndisp[b], sizeof(int)));
        if (c->lookahead && split) {
            // Split update: right section [cs, cend) (fixed width n2) and left
            // section [lrest, cs).  S_rs runs RS_R(j) then RS_L(j); S_tr runs
            // UPDATE_R(j) then UPDATE_L(j).  RS_L(j) overlaps UPDATE_R(j) and
            // RS_R(j+1) overlaps UPDATE_L(j).  Once the left section is used up the
            // right section is the whole rest (the paper's fallback).
            const int64_t cs = std::max(lrest, split_col);
            RsOut rsR, rsL;
            CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_panel[b], 0));
            CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_dgR, 0));
            if (E) CK(c, cudaEventRecord(E[0], c->s_rs));
            ST(rs_cols(c, c->s_rs, j, b, cs, cend, SEC_RIGHT, &rsR));
            CK(c, cudaEventRecord(c->ev_rsR, c->s_rs));
            CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_dgL, 0));
            ST(rs_cols(c, c->s_rs, j, b, lrest, cs, SEC_LEFT, &rsL));
            CK(c, cudaEventRecord(c->ev_rsL, c->s_rs));
            if (E) CK(c, cudaEventRecord(E[1], c->s_rs));
            CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_rsR, 0));
            ST(compute_cols(c, c->s_tr, j, b, cs, cend, rsR, true, false, E != nullptr));
            if (E) CK(c, cudaEventRecord(E[2], c->s_tr));
            CK(c, cudaEventRecord(c->ev_trsm, c->s_tr));
            ST(compute_cols(c, c->s_tr, j, b, cs, cend, rsR, false, true, E != nullptr));
            CK(c, cudaEventRecord(c->ev_dgR, c->s_tr));
            CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_rsL, 0));
            ST(compute_cols(c, c->s_tr, j, b, lrest, cs, rsL, true, true, E != nullptr));
            CK(c, cudaEventRecord(c->ev_dgL, c->s_tr));
            if (E) CK(c, cudaEventRecord(E[3], c->s_tr));
            CK(c, cudaEventRecord(c->ev_rest, c->s_tr));
            CK(c, cudaEventRecord(c->ev_next, c->s_tr));
        } else if (c->lookahead) {
            // RS + DTRSM of the rest on the high-priority S_rs (critical path),
            // only the long DGEMM at low priority on S_tr
            RsOut rs;
            CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_panel[b], 0));
            CK(c, cudaStreamWaitEvent(c->s_rs, c->ev_rest, 0));
            if (E) CK(c, cudaEventRecord(E[0], c->s_rs));
            ST(rs_cols(c, c->s_rs, j, b, lrest, cend, SEC_RIGHT, &rs));
            if (E) CK(c, cudaEventRecord(E[1], c->s_rs));
            ST(compute_cols(c, c->s_rs, j, b, lrest, cend, rs, true, false, E != nullptr));
            if (E) CK(c, cudaEventRecord(E[2], c->s_rs));
            CK(c, cudaEventRecord(c->ev_trsm, c->s_rs));
            CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_trsm, 0));
            ST(compute_cols(c, c->s_tr, j, b, lrest, cend, rs, false, true, E != nullptr));
            if (E) CK(c, cudaEventRecord(E[3], c->s_tr));
            CK(c, cudaEventRecord(c->ev_next, c->s_tr));
            CK(c, cudaEventRecord(c->ev_rest, c->s_tr));
        }
        if (c->lookahead) {
            if (E) CK(c, cudaEventRecord(E[4], c->s_la));
            if (own_next) ST(update_cols(c, c->s_la, j, b, lct, lct + jb1, SEC_LA));
            if (E) CK(c, cudaEventRecord(E[5], c->s_la));
            // FACT(j+1) competes for SMs: let the rest's LASWP + DTRSM (on the
            // critical path) finish first; FACT then overlaps the DGEMM.
            if (has_next) {
                CK(c, cudaStreamWaitEvent(c->s_la, c->ev_trsm, 0));
                ST(fact_panel(c, c->s_la, j + 1, bn, E ? E[7] : nullptr, E ? E[8] : nullptr));
                CK(c, cudaEventRecord(c->ev_panel[bn], c->s_la));
            }
            if (E) CK(c, cudaEventRecord(E[6], c->s_la));
            // la(j+1) touches panel j+2's columns: wait until rest(j) updated them
            CK(c, cudaStreamWaitEvent(c->s_la, c->ev_next, 0));
        } else {
            // no look-ahead (the baseline schedule): the whole update, then FACT(j+1)
            if (E) {
                CK(c, cudaEventRecord(E[0], c->s_la));
                CK(c, cudaEventRecord(E[4], c->s_la));
            }
            RsOut rs;
            ST(rs_cols(c, c->s_la, j, b, lct, cend, SEC_LA, &rs));
            if (E) CK(c, cudaEventRecord(E[1], c->s_la));
            ST(compute_cols(c, c->s_la, j, b, lct, cend, rs, true, false, E != nullptr));
            if (E) CK(c, cudaEventRecord(E[2], c->s_la));
            ST(compute_cols(c, c->s_la, j, b, lct, cend, rs, false, true, E != nullptr));
            if (E) {
                CK(c, cudaEventRecord(E[3], c->s_la));
                CK(c, cudaEventRecord(E[5], c->s_la));
            }
            if (has_next) ST(fact_panel(c, c->s_la, j + 1, bn, E ? E[7] : nullptr, E ? E[8] : nullptr));
            if (E) CK(c, cudaEventRecord(E[6], c->s_la));
        }
    }
    CK(c, cudaEventRecord(c->ev_rest, c->s_tr));
    CK(c, cudaStreamWaitEvent(c->s_la, c->ev_rest, 0));
    CK(c, cudaEventRecord(c->ev_rest, c->s_rs));
    CK(c, cudaStreamWaitEvent(c->s_la, c->ev_rest, 0));
    // the owner column saw the zero pivot: min over all ranks (unsigned: -1 = none)
    trace(c, "factor enqueued");
    ST(coll_allreduce(c, G_WORLD, c->fw.info, 1, COLL_MIN_U64, c->s_la));
    CK(c, cudaEventRecord(c->ev_t[1], c->s_la));
    std::vector<int> nd(c->timing ? nblk : 0, 0);
    if (c->timing) {
        CK(c, cudaMemcpyAsync(c->hstage, nd_hist, sizeof(int) * nblk, cudaMemcpyDeviceToHost,
                              c->s_la));
        CK(c, cudaFreeAsync(nd_hist, c->s_la));
    }
    CK(c, cudaStreamSynchronize(c->s_la));
    trace(c, "factor s_la synced");
    if (c->timing) std::memcpy(nd.data(), c->hstage, sizeof(int) * nblk);
    CK(c, cudaStreamSynchronize(c->s_tr));
    CK(c, cudaStreamSynchronize(c->s_rs));
    trace(c, "factor all synced");
    c->launches = t_launches - l0;
    c->factor_ms = ev_ms(c->ev_t[0], c->ev_t[1]);
    c->h2d_ms = c->h2d_last >= 0 ? ev_ms(c->ev_t[0], c->ev_arr[c->h2d_last]) : 0.0;
    c->pstart_ms = c->h2d_last >= 0 ? ev_ms(c->ev_t[0], c->ev_t[2]) : 0.0;
    if (c->h2d_last < 0) c->h2d_bytes = 0;
    c->timeline.clear();
    c->fact_detail.clear();
    c->dgemm_ms = c->laswp_ms = c->trsm_ms = c->fact_ms = 0;
    c->laswp_bytes = 0;
    if (c->timing) {
        c->timeline.reserve(6 * nblk);
        c->fact_detail.reserve(3 * nblk);
        for (int64_t j = 0; j < nblk; ++j) {
            if (j < jstart) {
                // a pipelined start's iterations ran per chunk without these
                // events (their records are a previous factorization's)
                for (int q = 0; q < 6; ++q) c->timeline.push_back(0.0);
                for (int q = 0; q < 3; ++q) c->fact_detail.push_back(0.0);
                continue;
            }
            cudaEvent_t *E = &c->tev[10 * j];
            const double rest_dg = ev_ms(E[2], E[3]);
            c->timeline.push_back(ev_ms(E[5], E[6]));
            c->timeline.push_back(ev_ms(E[4], E[5]));
            c->timeline.push_back(ev_ms(E[0], E[3]));
            c->timeline.push_back(ev_ms(E[0], E[1]));
            c->timeline.push_back(ev_ms(E[1], E[2]));
            c->timeline.push_back(rest_dg);
            c->dgemm_ms += rest_dg;
            c->laswp_ms += ev_ms(E[0], E[1]);
            c->trsm_ms += ev_ms(E[1], E[2]);
            // rest RS/LASWP of iteration j moves each gathered row and each
            // displaced row once over the rest's columns: read + write
            const int64_t j0 = j * c->NB, jb = jb_of(c, j);
            const bool own_next = j + 1 < nblk && c->mycol == (int)((j + 1) % c->Q);
            const int64_t lct = lcols_before(c, j0 + jb);
            const int64_t nrest = c->nloc - (lct + (own_next ? jb_of(c, j + 1) : 0));
            c->laswp_bytes += 2.0 * 8.0 * (double)(jb + nd[j]) * (double)std::max<int64_t>(nrest, 0);
            const bool nx = j + 1 < nblk;
            c->fact_detail.push_back(nx ? ev_ms(E[5], E[7]) : 0.0);
            c->fact_detail.push_back(nx ? ev_ms(E[7], E[8]) : 0.0);
            c->fact_detail.push_back(nx ? ev_ms(E[8], E[6]) : 0.0);
            if (nx) c->fact_ms += ev_ms(E[7], E[8]);
        }
    }
    ST(check_abort(c, c->s_la, "hpl_factor"));
    trace(c, "factor abort checked");
    int64_t info = -1;
    CK(c, cudaMemcpyAsync(c->hstage, c->fw.info, sizeof info, cudaMemcpyDeviceToHost, c->s_la));
    CK(c, cudaStreamSynchronize(c->s_la));
    std::memcpy(&info, c->hstage, sizeof info);
    trace(c, "factor end");
    c->state = hpl_ctx::S_FACTORED;
    if (info != -1) {
        c->singular = info;
        set_err(c, "exact zero pivot in global column %lld", (long long)info);
        return HPL_ERR_SINGULAR;
    }
    return HPL_OK;
}

}  // namespace

extern "C" {

hpl_status hpl_factor(hpl_ctx *c)
{
    if (!c) return HPL_ERR_ARG;
    if (!usable(c, hpl_ctx::S_INIT, "hpl_factor")) {
        if (c->state != hpl_ctx::S_BROKEN)
            set_err(c, "hpl_factor: context not in the initialised state");
        return HPL_ERR_STATE;
    }
    return factor_impl(c, nullptr);
}

hpl_status hpl_load_factor(hpl_ctx *c, const double *host, int64_t ld)
{
    if (!c || !host || ld < c->nloc) return HPL_ERR_ARG;
    if (c->state == hpl_ctx::S_BROKEN) return HPL_ERR_STATE;
    const int64_t nblk = cdiv(c->N, c->NB);
    if (c->nbuf < 4 || nblk < 2) {
        // (too few panel buffers for K >= 3 panels in flight: load, then
        // factor; nbuf is the same on every rank of a grid)
        ST(hpl_load_local(c, host, ld));
        return hpl_factor(c);
    }
    c->singular = -1;
    c->state = hpl_ctx::S_INIT;
    c->loaded = true;
    const Arrival a{host, ld};
    return factor_impl(c, &a);
}

hpl_status hpl_solve(hpl_ctx *c, double *x_host)
{
    if (!c) return HPL_ERR_ARG;
    if (!usable(c, hpl_ctx::S_FACTORED, "hpl_solve")) {
        if (c->state != hpl_ctx::S_BROKEN) set_err(c, "hpl_solve: call hpl_factor first");
        return HPL_ERR_STATE;
    }
    if (c->singular >= 0) return HPL_ERR_SINGULAR;
    CK(c, cudaSetDevice(c->device));
    const int64_t l0 = t_launches;
    trace(c, "solve start");
    CK(c, cudaEventRecord(c->ev_t[1], c->s_la));
    trace(c, "solve event recorded");
    {
        // Distributed block back substitution U x = y,
        // bottom block first, with a look-ahead.  Block row bb lives on
        // process row rb = bb mod P; its partial sums over the local columns
        // are split into FAR (column blocks >= bb+2, whose x is known one step
        // early) and NEAR (column block bb+1).  The far sums of block bb-2 run
        // on S_tr while S_la carries the critical chain of block bb: near
        // sums -> all-reduce over the process row -> diagonal solve on the
        // owner of block (bb, bb) -> broadcast of x_bb to every rank (x stays
        // replicated).  Partial buffers alternate by the parity of bb.  The far
        // sums run on the LOW-priority S_tr: the chain's kernels (the 16-CTA
        // cluster diagonal solve needs 16 free SMs of one GPC) get SMs first.
        const int64_t N = c->N, NB = c->NB, nblk = cdiv(N, NB);
        const int ycol = (int)((N / NB) % c->Q);            // owner of global column N
        const int64_t lcy = c->mycol == ycol ? lcols_before(c, N) : -1;
        const int64_t lcN = lcols_before(c, N);
        auto geom = [&](int64_t bb, int64_t *r0, int64_t *r1, int *nb, int64_t *farlo) {
            *r0 = bb * NB;
            *r1 = std::min<int64_t>(N, *r0 + NB);
            *nb = (int)(*r1 - *r0);
            *farlo = std::min<int64_t>(N, *r1 + NB);
        };
        // split count of the far sums: global sizes only, so the all-reduce
        // lines up on every rank of the process row
        auto sfar = [&](int64_t bb) {
            int64_t r0, r1, farlo;
            int nb;
            geom(bb, &r0, &r1, &nb, &farlo);
            return bs_splits(nb, 0, cdiv(cdiv(N - farlo, NB), c->Q) * NB, (int)NB);
        };
        auto tb = [&](int64_t bb) { return c->tbuf + (bb & 1) * (int64_t)17 * NB; };
        cudaEvent_t ev_far[2] = {c->ev_rsR, c->ev_rsL}, ev_x = c->ev_dgR;
        auto far = [&](int64_t bb) -> hpl_status {
            if (bb < 0) return HPL_OK;
            if (c->myrow == (int)(bb % c->P)) {
                int64_t r0, r1, farlo;
                int nb;
                geom(bb, &r0, &r1, &nb, &farlo);
                CK(c, bs_partial(c->s_tr, nb, c->A + lrows_before(c, r0) * c->lda, c->lda,
                                 lcols_before(c, farlo), lcN, (int)NB, c->Q, c->mycol, c->x, lcy,
                                 tb(bb), sfar(bb)));
            }
            CK(c, cudaEventRecord(ev_far[bb & 1], c->s_tr));
            return HPL_OK;
        };
        CK(c, cudaStreamWaitEvent(c->s_tr, c->ev_t[1], 0));
        ST(far(nblk - 1));
        ST(far(nblk - 2));
        for (int64_t bb = nblk - 1; bb >= 0; --bb) {
            int64_t r0, r1, farlo;
            int nb;
            geom(bb, &r0, &r1, &nb, &farlo);
            const int rb = (int)(bb % c->P), qb = (int)(bb % c->Q);
            if (c->myrow == rb) {
                if (bb == nblk - 1) trace(c, "solve first partial");
                const int64_t lr0 = lrows_before(c, r0);
                const int S = sfar(bb);
                double *Ubb = c->A + lr0 * c->lda + lcols_before(c, r0);
                if (c->Q == 1 && bs_diag_folds_near(nb)) {
                    // one process column: no row reduction, the near sums go into
                    // the diagonal solve (one launch per block on the chain)
                    CK(c, cudaStreamWaitEvent(c->s_la, ev_far[bb & 1], 0));
                    CK(c, bs_diag(c->s_la, nb, Ubb, c->lda, tb(bb), S, c->x + r0,
                                  (int)(farlo - r1), c->x + r1));
                } else {
                    CK(c, bs_partial(c->s_la, nb, c->A + lr0 * c->lda, c->lda, lcols_before(c, r1),
                                     lcols_before(c, farlo), (int)NB, c->Q, c->mycol, c->x, -1,
                                     tb(bb) + (int64_t)S * nb, 1));
                    CK(c, cudaStreamWaitEvent(c->s_la, ev_far[bb & 1], 0));
                    ST(coll_allreduce(c, G_ROW, tb(bb), (int64_t)(S + 1) * nb, COLL_SUM, c->s_la));
                    if (c->mycol == qb)
                        CK(c, bs_diag(c->s_la, nb, Ubb, c->lda, tb(bb), S + 1, c->x + r0));
                }
            } else {
                CK(c, cudaStreamWaitEvent(c->s_la, ev_far[bb & 1], 0));
            }
            ST(coll_bcast(c, G_WORLD, c->x + r0, sizeof(double) * nb, rb + qb * c->P, c->s_la));
            if (bb >= nblk - 2) trace(c, "solve block enqueued", bb);
            // x_bb is known everywhere: the far sums of block bb-2 may start
            CK(c, cudaEventRecord(ev_x, c->s_la));
            CK(c, cudaStreamWaitEvent(c->s_tr, ev_x, 0));
            ST(far(bb - 2));
        }
        CK(c, cudaEventRecord(ev_x, c->s_tr));
        CK(c, cudaStreamWaitEvent(c->s_la, ev_x, 0));
    }
    if (x_host)
        CK(c, cudaMemcpyAsync(c->hstage, c->x, sizeof(double) * c->N, cudaMemcpyDeviceToHost,
                              c->s_la));
    CK(c, cudaEventRecord(c->ev_t[2], c->s_la));
    trace(c, "solve enqueued");
    CK(c, cudaStreamSynchronize(c->s_la));
    trace(c, "solve synced");
    if (x_host) std::memcpy(x_host, c->hstage, sizeof(double) * c->N);
    ST(check_abort(c, c->s_la, "hpl_solve"));
    c->solve_ms = ev_ms(c->ev_t[1], c->ev_t[2]);
    c->launches += t_launches - l0;
    c->state = hpl_ctx::S_SOLVED;
    return HPL_OK;
}

hpl_status hpl_residual(hpl_ctx *c, double *resid)
{
    if (!c || !resid) return HPL_ERR_ARG;
    if (!usable(c, hpl_ctx::S_SOLVED, "hpl_residual")) {
        if (c->state != hpl_ctx::S_BROKEN) set_err(c, "hpl_residual: call hpl_solve first");
        return HPL_ERR_STATE;
    }
    if (c->loaded) {
        // the residual regenerates A0 and b0 from the seed; after
        // hpl_load_local the factored system is the caller's, not the seeded one
        set_err(c, "hpl_residual: the system came from hpl_load_local, not from the seed; "
                   "the seeded residual does not apply to it");
        return HPL_ERR_STATE;
    }
    CK(c, cudaSetDevice(c->device));
    // r and the row sums of |A0| for this process row's rows, summed over the
    // process row; the norms are then maxed over all ranks.
    CK(c, residual_partial(c->s_la, c->seed, c->N, c->NB, c->P, c->myrow, c->mloc, c->Q,
                           c->mycol, lcols_before(c, c->N), c->x, c->rvec, c->avec));
    ST(coll_allreduce(c, G_ROW, c->rvec, c->mloc, COLL_SUM, c->s_la));
    ST(coll_allreduce(c, G_ROW, c->avec, c->mloc, COLL_SUM, c->s_la));
    CK(c, residual_finalize(c->s_la, c->seed, c->N, c->NB, c->P, c->myrow, c->mloc, c->rvec,
                            c->avec, c->x, c->out4));
    ST(coll_allreduce(c, G_WORLD, c->out4, 4, COLL_MAX, c->s_la));
    double h[4];
    CK(c, cudaMemcpyAsync(c->hstage, c->out4, sizeof h, cudaMemcpyDeviceToHost, c->s_la));
    CK(c, cudaStreamSynchronize(c->s_la));
    std::memcpy(h, c->hstage, sizeof h);
    ST(check_abort(c, c->s_la, "hpl_residual"));
    *resid = scaled_residual(h, c->N);
    return HPL_OK;
}

hpl_status hpl_regenerate(hpl_ctx *c)
{
    if (!c || !c->A) return HPL_ERR_ARG;
    if (c->state == hpl_ctx::S_BROKEN) return HPL_ERR_STATE;
    c->singular = -1;
    return generate(c);
}

hpl_status hpl_load_local(hpl_ctx *c, const double *host, int64_t ld)
{
    if (!c || !host || ld < c->nloc) return HPL_ERR_ARG;
    if (c->state == hpl_ctx::S_BROKEN) return HPL_ERR_STATE;
    CK(c, cudaSetDevice(c->device));
    CK(c, cudaMemcpy2DAsync(c->A, c->lda * 8, host, ld * 8, c->nloc * 8, c->mloc,
                            cudaMemcpyHostToDevice, c->s_tr));
    CK(c, cudaStreamSynchronize(c->s_tr));
    c->singular = -1;
    c->state = hpl_ctx::S_INIT;
    c->loaded = true;
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
    for (int i = 0; i < c->trace_n; ++i)
        fprintf(stderr, "[hpl %.6f] rank %d %s %lld\n", (c->trace_t[i] % 1000000000000ll) * 1e-9,
                c->rank, c->trace_w[i], c->trace_k[i]);
    cudaSetDevice(c->device);
    for (cudaStream_t s : {c->s_la, c->s_tr, c->s_rs})
        if (s) cudaStreamSynchronize(s);
    release(c);
    delete c;
}

const char *hpl_last_error(const hpl_ctx *c) { return c ? c->err.c_str() : "null context"; }

int64_t hpl_singular_column(const hpl_ctx *c) { return c ? c->singular : -1; }

hpl_status hpl_get_ipiv(const hpl_ctx *c, int64_t *ipiv_host)
{
    if (!c || !ipiv_host) return HPL_ERR_ARG;
    if (c->state < hpl_ctx::S_FACTORED || c->state == hpl_ctx::S_BROKEN) return HPL_ERR_STATE;
    cudaSetDevice(c->device);
    if (cudaMemcpy(ipiv_host, c->gpiv, sizeof(int64_t) * c->N, cudaMemcpyDeviceToHost) !=
        cudaSuccess)
        return HPL_ERR_CUDA;
    return HPL_OK;
}

hpl_status hpl_get_local(const hpl_ctx *c, double *host, int64_t ld)
{
    if (!c || !host || ld < c->nloc) return HPL_ERR_ARG;
    cudaSetDevice(c->device);
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
    } else if (!strcmp(name, "gemm_cfg")) {
        if (value < -1 || value > 2) return HPL_ERR_ARG;
        c->gemm_cfg = c->fw.gemm_cfg = (int)value;
    } else if (!strcmp(name, "leaf_ctas")) {
        c->leaf_auto = false;
        c->fw.leaf_warp_ctas = 0;
        fact_set_leaf_ctas(&c->fw, (int)std::max<int64_t>(0, value), 0);
    } else if (!strcmp(name, "leaf_warp")) { c->leaf_auto = true; c->leaf_warp = (int)value; }
    else if (!strcmp(name, "leaf_few_ctas")) { c->leaf_auto = true; c->leaf_few_ctas = (int)value; }
    else if (!strcmp(name, "leaf_hide_ms")) { c->leaf_auto = true; c->leaf_hide_ms = (double)value; }
    else if (!strcmp(name, "leaf_cluster")) c->fw.leaf_cluster = value != 0;
    else if (!strcmp(name, "leaf_variant")) {
        if (value < 0 || value > 2) return HPL_ERR_ARG;
        c->fw.leaf_variant = (int)value;
    }
    else if (!strcmp(name, "split")) {
        if (value < 0 || value > 100) return HPL_ERR_ARG;
        c->split_pct = (int)value;
    }
    else if (!strcmp(name, "rs_peer")) c->rs_peer = value != 0 || c->P == 1;
    else if (!strcmp(name, "lb_peer")) c->lb_peer = value != 0 || c->Q == 1;
    else if (!strcmp(name, "coll_nccl")) c->coll_nccl = value != 0;
    else if (!strcmp(name, "fact_gather")) c->fact_gather_rows = std::max<int64_t>(0, value);
    else if (!strcmp(name, "fact_gather_ms")) c->fact_gather_ms = (double)value;
    else if (!strcmp(name, "peer_timeout_ms")) {
        if (value < 1) return HPL_ERR_ARG;
        c->fw.timeout_ns = (unsigned long long)value * 1000000ull;
    }
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
    out8[2] = lct;                             // look-ahead range begin
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

hpl_status hpl_debug_state(const hpl_ctx *c, uint64_t *out, int64_t cap)
{
    if (!c || !out || cap < 4 + N_GROUPS * MAX_GROUP + 2) return HPL_ERR_ARG;
    for (int gid = 0; gid < N_GROUPS; ++gid) out[gid] = c->g[gid].seq;
    uint64_t *fl = out + 4;
    if (c->cb) {
        cudaSetDevice(c->device);
        if (cudaMemcpy(fl, c->cb->flag, sizeof(c->cb->flag), cudaMemcpyDeviceToHost) != cudaSuccess)
            return HPL_ERR_CUDA;
    } else {
        std::memset(fl, 0, sizeof(uint64_t) * N_GROUPS * MAX_GROUP);
    }
    if (cudaMemcpy(fl + N_GROUPS * MAX_GROUP, c->fw.abort, 16, cudaMemcpyDeviceToHost) != cudaSuccess)
        return HPL_ERR_CUDA;
    return HPL_OK;
}

hpl_status hpl_phase_stats(const hpl_ctx *c, double *out10)   // 12 entries (hpl.h)
{
    if (!c || !out10) return HPL_ERR_ARG;
    double *out8 = out10;
    out10[8] = c->h2d_ms;
    out10[9] = c->h2d_bytes;
    out10[10] = c->pstart_ms;
    out10[11] = c->pstart_k;
    out8[0] = c->laswp_ms;
    out8[1] = c->laswp_bytes;
    out8[2] = c->trsm_ms;
    out8[3] = c->trsm_flop;
    out8[4] = c->fact_ms;
    out8[5] = c->solve_ms;
    // the back solve reads this rank's part of the upper triangle of U once
    // (plus y): sum over block rows of nb x (its local columns from the block on)
    double bytes = 0;
    const int64_t nblk = cdiv(c->N, c->NB);
    for (int64_t bb = 0; bb < nblk; ++bb) {
        if ((int)(bb % c->P) != c->myrow) continue;
        const int64_t r0 = bb * c->NB;
        const int64_t nb = std::min<int64_t>(c->NB, c->N - r0);
        bytes += 8.0 * (double)nb * (double)(lcols_before(c, c->N) - lcols_before(c, r0));
    }
    out8[6] = bytes;
    out8[7] = c->dgemm_ms;
    return HPL_OK;
}

}  // extern "C"
