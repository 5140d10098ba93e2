// hpl_ctx.cuh — the opaque hpl_ctx of include/hpl.h and the host-side
// helpers shared by hpl_comm.cu (process grid, peer memory, collectives) and
// hpl_driver.cu (the per-iteration schedule and the rest of the C ABI).
#pragma once
#include "hpl_internal.cuh"
#include "../../include/hpl.h"
#include <nccl.h>
#include <string>
#include <vector>

namespace hpl {

enum { G_WORLD = 0, G_ROW = 1, G_COL = 2, G_COLTR = 3 };

// A group of ranks (world / this process row / this process column).  The
// peer-memory transport (GroupDev, kernels_comm.cu) is always wired; the
// NCCL communicator exists only for a multi-process context.
struct Group {
    int size = 1, me = 0;
    int members[MAX_GROUP] = {};      // world ranks, member order
    ncclComm_t nccl = nullptr;
    unsigned long long seq = 0;       // barrier counter (identical on every member)
    GroupDev dev{};
};

// Panel buffers a context can hold (hpl_ctx::nbuf of them in use).
constexpr int MAX_PANELS = 8;

// Device pointers one rank shares with its peers (IPC handles in a
// multi-process grid, plain pointers in the single-device loopback).
struct PeerExports {
    double *A = nullptr;
    void *xbuf = nullptr;
    unsigned long long *rsflag = nullptr;
    double *panel[MAX_PANELS] = {};          // panel[b], b < nbuf (null beyond)
    unsigned long long *lbflag = nullptr;
    CommBlock *cb = nullptr;
};

}  // namespace hpl

struct hpl_ctx {
    // problem
    int64_t N = 0;
    int NB = 0, P = 1, Q = 1;
    uint64_t seed = 0;
    int rank = 0, nranks = 1, myrow = 0, mycol = 0, device = 0;
    bool dist = false;     // more than one rank
    bool loop = false;     // ranks are threads of this process on one device (loopback)
    // transport
    hpl::Group g[hpl::N_GROUPS];
    ncclComm_t world_nccl = nullptr;
    bool coll_nccl = false;           // option: NCCL for the non-hot collectives
    hpl::CommBlock *cb = nullptr;     // this rank's comm block
    std::vector<void *> ipc_open;     // peer mappings to close at free
    // P > 1: replicated top block, RS buffers (one set per section), pivot exchange
    double *Tbuf = nullptr;
    double *Ub[3] = {nullptr, nullptr, nullptr}, *Wb[3] = {nullptr, nullptr, nullptr};
    void *xbuf = nullptr;
    hpl::DistExchange xch{};
    unsigned long long xseq = 0;
    // P > 1 RS over peer memory (option rs_peer, default on)
    bool rs_peer = true;
    unsigned long long *rsflag = nullptr;
    hpl::RsPeers rsp{};
    unsigned long long rs_seq[3] = {0, 0, 0};
    // P > 1 gathered panel FACT for small panels
    const double *colpanel[hpl::MAX_P][hpl::MAX_PANELS] = {};
    double *Cp = nullptr;            // combined panel, cp_max_rows x NB (col-major)
    int64_t cp_max_rows = 0;
    int64_t fact_gather_rows = 65536;
    double fact_gather_ms = 8.0;
    unsigned long long fg_seq = 0;
    // Q > 1 LBCAST over peer memory (option lb_peer, default on).
    // lbflag[o] = last panel (+1) owner o has ready; lbflag[LB_DONE + q] = last
    // panel (+1) of this owner that column q copied.
    static constexpr int LB_DONE = 32;
    bool lb_peer = true;
    unsigned long long lb_base = 0, lb_next = 0;
    unsigned long long *lbflag = nullptr;
    std::vector<const double *> ppanel;         // [q * MAXBUF + b]: column q's panel[b]
    std::vector<unsigned long long *> pflag;    // [q]: column q's lbflag
    double *rvec = nullptr, *avec = nullptr, *bvec = nullptr;   // residual partial sums
    // local storage
    int64_t mloc = 0, nloc = 0, lda = 0;
    double *A = nullptr;
    // per-panel state (panel, L11^{-1}, pivot plan): panels j, j+1, j+2 are
    // live at once in the look-ahead loop, so NBUF = 3 buffers suffice; a
    // context keeps MAXBUF (memory permitting) so hpl_load_factor's pipelined
    // start can have K + 1 panels in flight.  nbuf = buffers in use, the same
    // on every rank of a grid (peers index each other's buffer j mod nbuf:
    // the LBCAST pull, the gathered FACT).
    static constexpr int NBUF = 3, MAXBUF = hpl::MAX_PANELS;
    int nbuf = NBUF;
    double *panel[MAXBUF] = {};
    int64_t ldp = 0;
    double *linv[MAXBUF] = {};
    int64_t ldlinv = 0;
    int64_t *src[MAXBUF] = {};
    int64_t *disp[MAXBUF] = {};
    int *ndisp[MAXBUF] = {};
    int64_t *gpiv = nullptr;
    double *U = nullptr;     // gathered block rows (pre-DTRSM), NB x ldu
    double *U2 = nullptr;    // L11^{-1} U (the DGEMM's B operand), NB x ldu
    int64_t ldu = 0;
    double *scratch = nullptr;
    double *x = nullptr, *tbuf = nullptr, *out4 = nullptr;
    // pinned host staging (N doubles, at least 16): device->host results are
    // copied here asynchronously, the stream is synchronised, then the caller's
    // buffer is filled on the host.  A pageable copy queued behind waits on
    // other ranks would block inside the driver while other threads (loopback
    // ranks) need it to launch the work those waits depend on.
    double *hstage = nullptr;
    hpl::FactWork fw{};
    cudaStream_t s_la = nullptr, s_tr = nullptr, s_rs = nullptr;
    cudaEvent_t ev_panel[MAXBUF] = {}, ev_rest = nullptr;
    // hpl_load_factor's pipelined start: copy stream and one arrival event
    // per column chunk (created on first use)
    cudaStream_t s_h2d = nullptr;
    std::vector<cudaEvent_t> ev_arr;
    cudaEvent_t ev_next = nullptr;   // rest(j) has updated panel j+2's columns
    cudaEvent_t ev_trsm = nullptr;   // rest(j)'s LASWP+DTRSM done: FACT(j+1) may start
    cudaEvent_t ev_rsR = nullptr, ev_rsL = nullptr, ev_dgR = nullptr, ev_dgL = nullptr;
    // options
    int split_pct = 0;               // split update: right-section share
    bool lookahead = true;
    int nbmin = 16;
    int gemm_cfg = -1;
    bool leaf_auto = true;           // adaptive leaf grid (fact_panel)
    int leaf_few_ctas = 8;
    int leaf_warp = 0;               // >0: hidden FACT uses up to this many one-warp leaf CTAs
    double leaf_hide_ms = 15.0;
    bool timing = false;
    std::vector<cudaEvent_t> tev;   // 10 events per iteration when timing
    std::vector<double> timeline;   // 6 values per iteration (ms)
    std::vector<double> fact_detail;  // 3 values per iteration (ms)
    cudaEvent_t ev_t[3] = {nullptr, nullptr, nullptr};  // factor start/end, solve end
    double factor_ms = 0, solve_ms = 0;
    double dgemm_ms = 0, dgemm_flop = 0;   // trailing (rest) DGEMM launches, timing on
    int64_t dgemm_launches = 0;
    double laswp_ms = 0, laswp_bytes = 0;  // rest RS/LASWP phases, timing on
    double trsm_ms = 0, trsm_flop = 0;     // rest DTRSM phases, timing on
    double fact_ms = 0;                    // FACT(j+1) proper, summed, timing on
    double h2d_ms = 0, h2d_bytes = 0;      // hpl_load_factor: factor start -> last chunk landed
    int h2d_last = -1;
    double pstart_ms = 0;                  // factor start -> end of the pipelined start
    int pstart_k = 0;                      // iterations in the pipelined start
    // state
    enum { S_NONE, S_INIT, S_FACTORED, S_SOLVED, S_BROKEN } state = S_NONE;
    bool loaded = false;             // [A | b] came from hpl_load_local (not the seeded system)
    std::string err;
    int64_t singular = -1;
    int64_t launches = 0;
    // HPL_TRACE diagnostics (hpl_driver.cu trace())
    long long trace_t[64] = {};
    const char *trace_w[64] = {};
    long long trace_k[64] = {};
    int trace_n = 0;
};

namespace hpl {

void set_err(hpl_ctx *c, const char *fmt, ...);

#define CK(ctx, expr)                                                                       \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess) {                                                            \
            hpl::set_err(ctx, "%s:%d %s -> %s", __FILE__, __LINE__, #expr,                  \
                         cudaGetErrorString(_e));                                           \
            return HPL_ERR_CUDA;                                                            \
        }                                                                                   \
    } while (0)

#define NK(ctx, expr)                                                                       \
    do {                                                                                    \
        ncclResult_t _r = (expr);                                                           \
        if (_r != ncclSuccess) {                                                            \
            hpl::set_err(ctx, "%s:%d %s -> %s", __FILE__, __LINE__, #expr,                  \
                         ncclGetErrorString(_r));                                           \
            return HPL_ERR_NCCL;                                                            \
        }                                                                                   \
    } while (0)

#define ST(expr)                                \
    do {                                        \
        hpl_status _s = (expr);                 \
        if (_s != HPL_OK) return _s;            \
    } while (0)

// numroc: number of indices of an extent-n dimension owned by coordinate me
inline int64_t numroc(int64_t n, int nb, int me, int nprocs)
{
    const int64_t nblocks = n / nb;
    int64_t cnt = (nblocks / nprocs) * nb;
    const int64_t extra = nblocks % nprocs;
    if (me < extra) cnt += nb;
    else if (me == extra) cnt += n % nb;
    return cnt;
}

// ---- hpl_comm.cu
// Allocate the context's device memory, streams and events (P, Q, rank set).
hpl_status alloc_ctx(hpl_ctx *c);
// Panel buffers: how many this device can hold for `copies` contexts, and
// allocate buffers [nbuf, n).
int panels_wanted(hpl_ctx *c, int copies);
hpl_status grow_panels(hpl_ctx *c, int n);
// Wire the peer tables (RS, pivot exchange, gathered FACT, LBCAST, groups)
// from every rank's exports (world-indexed, this process's address space).
hpl_status setup_peers(hpl_ctx *c, const std::vector<PeerExports> &ex);
PeerExports exports_of(const hpl_ctx *c);
// Collectives over group gid (member indices; root = member index).
hpl_status coll_bcast(hpl_ctx *c, int gid, void *buf, size_t bytes, int root, cudaStream_t st);
hpl_status coll_allreduce(hpl_ctx *c, int gid, void *buf, int64_t n, int op, cudaStream_t st);
// Flag barrier over group gid.
hpl_status coll_barrier(hpl_ctx *c, int gid, cudaStream_t st);
// Device-to-device copies of the schedule: the copy engine for a
// multi-process rank, SMs in a loopback (the ranks' copies then never queue
// behind one another on a shared engine while their kernels wait on each other).
hpl_status d2d(hpl_ctx *c, cudaStream_t st, void *dst, const void *src, size_t bytes);
hpl_status d2d_2d(hpl_ctx *c, cudaStream_t st, void *dst, size_t dpitch, const void *src,
                  size_t spitch, size_t width, size_t rows);
void release(hpl_ctx *c);
hpl_status generate(hpl_ctx *c);
// HPL_ERR_PEER (and the broken state) if a bounded wait of this context gave up.
hpl_status check_abort(hpl_ctx *c, cudaStream_t st, const char *where);
SpinCtl spin(const hpl_ctx *c);

}  // namespace hpl
