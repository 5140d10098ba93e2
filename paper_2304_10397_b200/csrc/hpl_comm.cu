// hpl_comm.cu — process grid, peer memory and collectives of libhpl.so.
//
// One rank per GPU, 2D block-cyclic over P x Q with
// rank = p + q*P.  The exchanges of the method run over peer
// memory: the RS row gather (rs_gather_peer), the pivot search
// across the process column (the distributed leaf), the panel
// LBCAST along the process row (copy-engine pulls) and the
// remaining small collectives (kernels_comm.cu).  Where the peers' memory
// comes from is the only thing that differs between the two multi-rank modes:
//
//  - hpl_init_dist: one process per GPU; every rank exports its buffers as
//    CUDA IPC handles, all-gathered over NCCL once at init; NCCL
//    communicators also carry the optional NCCL variants (rs_peer=0,
//    lb_peer=0, coll_nccl=1);
//  - hpl_init_loopback: all P*Q ranks are contexts of ONE process on ONE
//    device, driven by one host thread each ("ranks are
//    concurrent workers in one process"); the peer tables hold the sibling
//    contexts' plain device pointers and no NCCL is involved.  The same
//    kernels, flags and schedule run as on P*Q GPUs, so the single-GPU test
//    box checks the multi-GPU data path against the oracle.
#include "hpl_ctx.cuh"
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace hpl {

void set_err(hpl_ctx *c, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
}

SpinCtl spin(const hpl_ctx *c) { return c->fw.spin(); }

hpl_status check_abort(hpl_ctx *c, cudaStream_t st, const char *where)
{
    unsigned long long ab[2] = {0, 0};
    CK(c, cudaMemcpyAsync(c->hstage, c->fw.abort, sizeof ab, cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    std::memcpy(ab, c->hstage, sizeof ab);
    const unsigned long long code = ab[0];
    if (code == 0) return HPL_OK;
    static const char *site[] = {"?", "FACT grid barrier", "pivot exchange with the process column",
                                 "pivot winner flag", "RS barrier", "LBCAST flag",
                                 "group barrier (collective)"};
    const unsigned s = (unsigned)(code & 15);
    set_err(c, "%s: rank %d: a peer-memory wait timed out at the %s (site %u, slot/group %llu, "
               "lane/member %llu, expected %llu, saw %llu): a peer rank failed or did not take "
               "part; the context must be freed", where, c->rank, site[s < 7 ? s : 0], s,
            (code >> 4) & 15, code >> 8, ab[1] >> 32, ab[1] & 0xffffffffull);
    c->state = hpl_ctx::S_BROKEN;
    return HPL_ERR_PEER;
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
    ST(grow_panels(c, hpl_ctx::NBUF));
    if (!M((void **)&c->gpiv, sizeof(int64_t) * (size_t)c->N)) return HPL_ERR_OOM;
    if (!M((void **)&c->U, sizeof(double) * NBs * c->ldu)) return HPL_ERR_OOM;
    if (!M((void **)&c->U2, sizeof(double) * NBs * c->ldu)) return HPL_ERR_OOM;
    if (!M((void **)&c->scratch, sizeof(double) * round_up(NBs, 16) * NBs)) return HPL_ERR_OOM;
    if (!M((void **)&c->x, sizeof(double) * (size_t)c->N)) return HPL_ERR_OOM;
    // back-solve partial sums: 2 parities x (<= 16 far shares + 1 near share) x NB
    if (!M((void **)&c->tbuf, sizeof(double) * 2 * 17 * NBs)) return HPL_ERR_OOM;
    if (!M((void **)&c->out4, sizeof(double) * 4)) return HPL_ERR_OOM;
    if (cudaMallocHost((void **)&c->hstage, sizeof(double) * (size_t)std::max<int64_t>(c->N, 16)) !=
        cudaSuccess) {
        cudaGetLastError();
        set_err(c, "cudaMallocHost of the %lld-double staging buffer failed", (long long)c->N);
        return HPL_ERR_OOM;
    }
    const size_t mrow = sizeof(double) * (size_t)std::max<int64_t>(c->mloc, 1);
    if (!M((void **)&c->rvec, mrow) || !M((void **)&c->avec, mrow) || !M((void **)&c->bvec, mrow))
        return HPL_ERR_OOM;
    if (c->P > 1) {
        const size_t rs = sizeof(double) * NBs * (size_t)round_up(c->nloc, 16);
        if (!M((void **)&c->Tbuf, sizeof(double) * NBs * NBs)) return HPL_ERR_OOM;
        for (int k = 0; k < 3; ++k) {
            if (!M((void **)&c->Ub[k], rs)) return HPL_ERR_OOM;
            if (!M((void **)&c->Wb[k], rs)) return HPL_ERR_OOM;
        }
        // pivot-exchange area: 2 parities x P records of (2 + NB) doubles, then 2P flags
        const size_t rec_bytes = sizeof(double) * 2 * (size_t)c->P * (2 + NBs);
        const size_t xbytes = rec_bytes + sizeof(unsigned long long) * 2 * c->P;
        if (!M(&c->xbuf, xbytes)) return HPL_ERR_OOM;
        CK(c, cudaMemset(c->xbuf, 0, xbytes));
        const size_t fbytes = sizeof(unsigned long long) * RS_SLOTS * MAX_P;
        if (!M((void **)&c->rsflag, fbytes)) return HPL_ERR_OOM;
        CK(c, cudaMemset(c->rsflag, 0, fbytes));
        // combined panel for the gathered FACT: up to 64 Ki global rows
        c->cp_max_rows = std::min<int64_t>(c->N, (int64_t)1 << 16);
        if (!M((void **)&c->Cp, sizeof(double) * (size_t)round_up(c->cp_max_rows, 16) * NBs))
            return HPL_ERR_OOM;
    }
    if (c->Q > 1) {
        const size_t fbytes = sizeof(unsigned long long) * 64;
        if (!M((void **)&c->lbflag, fbytes)) return HPL_ERR_OOM;
        CK(c, cudaMemset(c->lbflag, 0, fbytes));
    }
    if (c->nranks > 1) {
        if (!M((void **)&c->cb, sizeof(CommBlock))) return HPL_ERR_OOM;
        CK(c, cudaMemset(c->cb->flag, 0, sizeof(c->cb->flag)));
    }
    CK(c, fact_work_alloc(&c->fw));
    CK(c, dgemm_prepare());
    CK(c, fact_prepare());
    CK(c, solve_prepare());
    if (c->loop) {
        // every rank's cooperative leaf must fit on the device at once (the
        // P leaves of a column wait on each other): a share of the SMs each
        int sms = 148;
        CK(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
        c->fw.max_ctas = std::max(1, sms / c->nranks);
        c->fw.timeout_ns = 20ull * 1000000000ull;
        c->fw.plain_launch = 1;
    }
    int lo, hi;
    CK(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(c, cudaStreamCreateWithPriority(&c->s_la, cudaStreamNonBlocking, hi));
    CK(c, cudaStreamCreateWithPriority(&c->s_tr, cudaStreamNonBlocking, lo));
    CK(c, cudaStreamCreateWithPriority(&c->s_rs, cudaStreamNonBlocking, hi));
    for (cudaEvent_t *e : {&c->ev_rsR, &c->ev_rsL, &c->ev_dgR, &c->ev_dgL, &c->ev_next,
                           &c->ev_rest, &c->ev_trsm})
        CK(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (int k = 0; k < 3; ++k) CK(c, cudaEventCreate(&c->ev_t[k]));
    // one rank: more panel buffers right away (several ranks agree first)
    if (c->nranks == 1) ST(grow_panels(c, panels_wanted(c, 1)));
    return HPL_OK;
}

int panels_wanted(hpl_ctx *c, int copies)
{
    // MAXBUF panel states if they leave >= 4 GB free (copies: contexts on
    // this device that grow alike — the loopback's ranks)
    const size_t NBs = (size_t)c->NB;
    const size_t per = sizeof(double) * ((size_t)c->ldp * (NBs + 1) + (size_t)c->ldlinv * NBs);
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return c->nbuf;
    }
    const size_t need = (size_t)copies * per * (size_t)(hpl_ctx::MAXBUF - c->nbuf);
    return fr > need + ((size_t)4 << 30) ? hpl_ctx::MAXBUF : c->nbuf;
}

hpl_status grow_panels(hpl_ctx *c, int nbuf)
{
    const size_t NBs = (size_t)c->NB;
    const size_t pbytes = sizeof(double) * (size_t)c->ldp * (NBs + 1);
    for (int b = 0; b < nbuf; ++b) {
        if (c->panel[b]) continue;
        bool ok = cudaMalloc((void **)&c->panel[b], pbytes) == cudaSuccess &&
                  cudaMalloc((void **)&c->linv[b], sizeof(double) * (size_t)c->ldlinv * NBs) ==
                      cudaSuccess &&
                  cudaMalloc((void **)&c->src[b], sizeof(int64_t) * NBs) == cudaSuccess &&
                  cudaMalloc((void **)&c->disp[b], sizeof(int64_t) * 2 * NBs) == cudaSuccess &&
                  cudaMalloc((void **)&c->ndisp[b], sizeof(int)) == cudaSuccess;
        if (!ok) {
            cudaGetLastError();
            set_err(c, "cudaMalloc of panel buffer %d failed", b);
            return HPL_ERR_OOM;
        }
        CK(c, cudaMemset(c->panel[b], 0, pbytes));
        CK(c, cudaEventCreateWithFlags(&c->ev_panel[b], cudaEventDisableTiming));
    }
    c->nbuf = std::max(c->nbuf, nbuf);
    return HPL_OK;
}

PeerExports exports_of(const hpl_ctx *c)
{
    PeerExports e;
    e.A = c->A;
    e.xbuf = c->xbuf;
    e.rsflag = c->rsflag;
    for (int b = 0; b < c->nbuf; ++b) e.panel[b] = c->panel[b];
    e.lbflag = c->lbflag;
    e.cb = c->cb;
    return e;
}

hpl_status setup_peers(hpl_ctx *c, const std::vector<PeerExports> &ex)
{
    const int P = c->P, Q = c->Q, MB = hpl_ctx::MAXBUF;
    if ((int)ex.size() != c->nranks) return HPL_ERR_ARG;
    if (P > 1) {
        c->rsp.P = P;
        c->rsp.myrow = c->myrow;
        c->rsp.my_flag = c->rsflag;
        const size_t rec_bytes = sizeof(double) * 2 * (size_t)P * (2 + c->NB);
        c->xch.P = P;
        c->xch.myrow = c->myrow;
        c->xch.recd = 2 + c->NB;
        for (int p = 0; p < P; ++p) {
            const PeerExports &e = ex[p + c->mycol * P];
            c->rsp.A[p] = e.A;
            c->rsp.flag[p] = e.rsflag;
            for (int b = 0; b < MB; ++b) c->colpanel[p][b] = e.panel[b];
            c->xch.rec[p] = static_cast<double *>(e.xbuf);
            c->xch.flag[p] = reinterpret_cast<unsigned long long *>(static_cast<char *>(e.xbuf) +
                                                                    rec_bytes);
        }
        c->xch.my_rec = c->xch.rec[c->myrow];
        c->xch.my_flag = c->xch.flag[c->myrow];
    }
    if (Q > 1) {
        c->ppanel.assign((size_t)Q * MB, nullptr);
        c->pflag.assign(Q, nullptr);
        for (int q = 0; q < Q; ++q) {
            const PeerExports &e = ex[c->myrow + q * P];
            for (int b = 0; b < MB; ++b) c->ppanel[(size_t)q * MB + b] = e.panel[b];
            c->pflag[q] = e.lbflag;
        }
    }
    for (int gid = 0; gid < N_GROUPS; ++gid) {
        Group &g = c->g[gid];
        if (gid == G_WORLD) {
            g.size = c->nranks;
            g.me = c->rank;
            for (int r = 0; r < c->nranks; ++r) g.members[r] = r;
        } else if (gid == G_ROW) {
            g.size = Q;
            g.me = c->mycol;
            for (int q = 0; q < Q; ++q) g.members[q] = c->myrow + q * P;
        } else {
            g.size = P;
            g.me = c->myrow;
            for (int p = 0; p < P; ++p) g.members[p] = p + c->mycol * P;
        }
        g.dev.size = g.size;
        g.dev.me = g.me;
        g.dev.gid = gid;
        for (int m = 0; m < g.size; ++m) g.dev.blk[m] = ex[g.members[m]].cb;
    }
    return HPL_OK;
}

hpl_status d2d(hpl_ctx *c, cudaStream_t st, void *dst, const void *src, size_t bytes)
{
    return d2d_2d(c, st, dst, bytes, src, bytes, bytes, 1);
}

hpl_status d2d_2d(hpl_ctx *c, cudaStream_t st, void *dst, size_t dpitch, const void *src,
                  size_t spitch, size_t width, size_t rows)
{
    if (c->loop)
        CK(c, copy2d_sm(st, dst, (int64_t)dpitch, src, (int64_t)spitch, (int64_t)width,
                        (int64_t)rows));
    else
        CK(c, cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToDevice,
                                st));
    return HPL_OK;
}

// ---------------------------------------------------------------- collectives
hpl_status coll_barrier(hpl_ctx *c, int gid, cudaStream_t st)
{
    Group &g = c->g[gid];
    if (g.size <= 1) return HPL_OK;
    CK(c, group_barrier(st, g.dev, ++g.seq, spin(c)));
    return HPL_OK;
}

static ncclDataType_t nccl_type(int op) { return op == COLL_MIN_U64 ? ncclUint64 : ncclDouble; }
static ncclRedOp_t nccl_op(int op)
{
    return op == COLL_SUM ? ncclSum : op == COLL_MAX ? ncclMax : ncclMin;
}

hpl_status coll_bcast(hpl_ctx *c, int gid, void *buf, size_t bytes, int root, cudaStream_t st)
{
    Group &g = c->g[gid];
    if (g.size <= 1 || bytes == 0) return HPL_OK;
    if (c->coll_nccl && g.nccl) {
        NK(c, ncclBroadcast(buf, buf, bytes, ncclChar, root, g.nccl, st));
        return HPL_OK;
    }
    const size_t chunk = sizeof(double) * (size_t)STAGE_DOUBLES;
    for (size_t off = 0; off < bytes; off += chunk) {
        const size_t n = std::min(chunk, bytes - off);
        char *p = static_cast<char *>(buf) + off;
        if (g.me == root)
            ST(d2d(c, st, c->cb->stage[gid], p, n));
        ST(coll_barrier(c, gid, st));
        if (g.me != root)
            ST(d2d(c, st, p, g.dev.blk[root]->stage[gid], n));
        ST(coll_barrier(c, gid, st));
    }
    return HPL_OK;
}

hpl_status coll_allreduce(hpl_ctx *c, int gid, void *buf, int64_t n, int op, cudaStream_t st)
{
    Group &g = c->g[gid];
    if (g.size <= 1 || n <= 0) return HPL_OK;
    if (c->coll_nccl && g.nccl) {
        NK(c, ncclAllReduce(buf, buf, (size_t)n, nccl_type(op), nccl_op(op), g.nccl, st));
        return HPL_OK;
    }
    for (int64_t off = 0; off < n; off += STAGE_DOUBLES) {
        const int64_t k = std::min<int64_t>(STAGE_DOUBLES, n - off);
        char *p = static_cast<char *>(buf) + 8 * off;
        ST(d2d(c, st, c->cb->stage[gid], p, 8 * (size_t)k));
        ST(coll_barrier(c, gid, st));
        CK(c, group_reduce(st, g.dev, op, k, p));
        ST(coll_barrier(c, gid, st));
    }
    return HPL_OK;
}

hpl_status generate(hpl_ctx *c)
{
    CK(c, cudaSetDevice(c->device));
    CK(c, gen_local(c->s_tr, c->seed, c->N, c->NB, c->P, c->Q, c->myrow, c->mycol, c->mloc,
                    c->nloc, c->A, c->lda));
    CK(c, cudaStreamSynchronize(c->s_tr));
    c->state = hpl_ctx::S_INIT;
    c->loaded = false;
    return HPL_OK;
}

void release(hpl_ctx *c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    cudaFree(c->A);
    for (int b = 0; b < hpl_ctx::MAXBUF; ++b) {
        cudaFree(c->panel[b]); cudaFree(c->linv[b]);
        cudaFree(c->src[b]); cudaFree(c->disp[b]); cudaFree(c->ndisp[b]);
        if (c->ev_panel[b]) cudaEventDestroy(c->ev_panel[b]);
    }
    cudaFree(c->gpiv); cudaFree(c->U); cudaFree(c->U2); cudaFree(c->scratch);
    cudaFree(c->x); cudaFree(c->tbuf); cudaFree(c->out4);
    cudaFreeHost(c->hstage);
    cudaFree(c->rvec); cudaFree(c->avec); cudaFree(c->bvec);
    cudaFree(c->Tbuf);
    for (int k = 0; k < 3; ++k) { cudaFree(c->Ub[k]); cudaFree(c->Wb[k]); }
    for (void *pp : c->ipc_open) cudaIpcCloseMemHandle(pp);
    cudaFree(c->Cp);
    cudaFree(c->lbflag);
    cudaFree(c->rsflag);
    cudaFree(c->xbuf);
    cudaFree(c->cb);
    for (int gid = 0; gid < N_GROUPS; ++gid)
        if (c->g[gid].nccl) ncclCommDestroy(c->g[gid].nccl);
    if (c->world_nccl) ncclCommDestroy(c->world_nccl);
    fact_work_free(&c->fw);
    for (cudaEvent_t e : {c->ev_rest, c->ev_trsm, c->ev_next, c->ev_rsR, c->ev_rsL, c->ev_dgR,
                          c->ev_dgL})
        if (e) cudaEventDestroy(e);
    for (auto e : c->tev) cudaEventDestroy(e);
    for (int k = 0; k < 3; ++k)
        if (c->ev_t[k]) cudaEventDestroy(c->ev_t[k]);
    for (cudaStream_t s : {c->s_la, c->s_tr, c->s_rs, c->s_h2d})
        if (s) cudaStreamDestroy(s);
    for (cudaEvent_t e : c->ev_arr) cudaEventDestroy(e);
}

namespace {

// Multi-process: every rank's exports travel as CUDA IPC handles (one NCCL
// all-gather over the world at init); a rank maps what its exchanges read —
// the process column's A, RS flags, pivot-exchange areas and packed panels,
// the process row's panel buffers and LBCAST flags, everyone's comm block.
constexpr int HP = 3;                   // handle index of panel[0]
constexpr int NH = HP + MAX_PANELS + 2;  // A, xbuf, rsflag, panel[0..MAX_PANELS), lbflag, cb
struct Handles {
    cudaIpcMemHandle_t h[NH];
    int have[NH];
};

hpl_status exchange_ipc(hpl_ctx *c, std::vector<PeerExports> *out)
{
    const PeerExports me = exports_of(c);
    void *ptrs[NH] = {me.A, me.xbuf, me.rsflag};
    for (int b = 0; b < MAX_PANELS; ++b) ptrs[HP + b] = me.panel[b];
    ptrs[HP + MAX_PANELS] = me.lbflag;
    ptrs[HP + MAX_PANELS + 1] = me.cb;
    Handles mine{};
    for (int k = 0; k < NH; ++k) {
        mine.have[k] = ptrs[k] != nullptr;
        if (ptrs[k]) CK(c, cudaIpcGetMemHandle(&mine.h[k], ptrs[k]));
    }
    char *dh = nullptr;
    CK(c, cudaMalloc(&dh, sizeof(Handles) * c->nranks));
    CK(c, cudaMemcpy(dh + sizeof(Handles) * c->rank, &mine, sizeof mine, cudaMemcpyHostToDevice));
    NK(c, ncclAllGather(dh + sizeof(Handles) * c->rank, dh, sizeof(Handles), ncclChar,
                        c->world_nccl, c->s_la));
    CK(c, cudaStreamSynchronize(c->s_la));
    std::vector<Handles> all(c->nranks);
    CK(c, cudaMemcpy(all.data(), dh, sizeof(Handles) * c->nranks, cudaMemcpyDeviceToHost));
    cudaFree(dh);
    out->assign(c->nranks, PeerExports{});
    (*out)[c->rank] = me;
    for (int r = 0; r < c->nranks; ++r) {
        if (r == c->rank) continue;
        const bool same_col = r / c->P == c->mycol, same_row = r % c->P == c->myrow;
        auto open = [&](int k) -> void * {
            if (!all[r].have[k]) return nullptr;
            void *p = nullptr;
            if (cudaIpcOpenMemHandle(&p, all[r].h[k], cudaIpcMemLazyEnablePeerAccess) !=
                cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
            c->ipc_open.push_back(p);
            return p;
        };
        PeerExports &e = (*out)[r];
        if (same_col) {
            e.A = static_cast<double *>(open(0));
            e.xbuf = open(1);
            e.rsflag = static_cast<unsigned long long *>(open(2));
            if (!e.A || !e.xbuf || !e.rsflag) goto fail;
        }
        if (same_col || same_row) {
            // every rank holds the same nbuf buffers (agreed at init)
            for (int b = 0; b < c->nbuf; ++b)
                if (!(e.panel[b] = static_cast<double *>(open(HP + b)))) goto fail;
        }
        if (same_row && c->Q > 1 &&
            !(e.lbflag = static_cast<unsigned long long *>(open(HP + MAX_PANELS))))
            goto fail;
        if (!(e.cb = static_cast<CommBlock *>(open(HP + MAX_PANELS + 1)))) goto fail;
        continue;
    fail:
        set_err(c, "cudaIpcOpenMemHandle of rank %d's buffers failed (ranks must share one node "
                   "with peer access)", r);
        return HPL_ERR_CUDA;
    }
    return HPL_OK;
}

hpl_status check_args(int64_t N, int32_t NB, int32_t P, int32_t Q)
{
    if (N < 1 || NB < 1 || NB > N || P < 1 || Q < 1) return HPL_ERR_ARG;
    // implementation limits, reading A18 (listed in include/hpl.h)
    if (NB > 1024 || (NB & 1) || N >= (int64_t)1 << 31) return HPL_ERR_ARG;
    if (P > MAX_P || Q > 32 || P * Q > MAX_GROUP) return HPL_ERR_ARG;
    return HPL_OK;
}

}  // namespace

}  // namespace hpl

using namespace hpl;

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
    if (s == HPL_OK) s = setup_peers(c, std::vector<PeerExports>(1, exports_of(c)));
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
    hpl_ctx *c = new hpl_ctx();
    *out = c;
    c->N = N; c->NB = NB; c->P = P; c->Q = Q; c->seed = seed;
    c->rank = rank; c->nranks = nranks; c->myrow = rank % P; c->mycol = rank / P;
    c->device = device;
    c->dist = nranks > 1;
    CK(c, cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof id);
    NK(c, ncclCommInitRank(&c->world_nccl, nranks, id, rank));
    NK(c, ncclCommSplit(c->world_nccl, 0, rank, &c->g[G_WORLD].nccl, nullptr));
    NK(c, ncclCommSplit(c->world_nccl, c->myrow, c->mycol, &c->g[G_ROW].nccl, nullptr));
    NK(c, ncclCommSplit(c->world_nccl, c->mycol, c->myrow, &c->g[G_COL].nccl, nullptr));
    NK(c, ncclCommSplit(c->world_nccl, c->mycol, c->myrow, &c->g[G_COLTR].nccl, nullptr));
    ST(alloc_ctx(c));
    if (nranks > 1) {
        // the same number of panel buffers on every rank: the minimum wanted
        const int32_t want = panels_wanted(c, 1);
        int32_t *d = reinterpret_cast<int32_t *>(c->out4);
        CK(c, cudaMemcpy(d, &want, sizeof want, cudaMemcpyHostToDevice));
        NK(c, ncclAllReduce(d, d, 1, ncclInt32, ncclMin, c->world_nccl, c->s_la));
        int32_t agreed = 0;
        CK(c, cudaMemcpyAsync(&agreed, d, sizeof agreed, cudaMemcpyDeviceToHost, c->s_la));
        CK(c, cudaStreamSynchronize(c->s_la));
        ST(grow_panels(c, agreed));
    }
    std::vector<PeerExports> ex;
    if (nranks > 1) ST(exchange_ipc(c, &ex));
    else ex.assign(1, exports_of(c));
    ST(setup_peers(c, ex));
    return generate(c);
}

hpl_status hpl_init_loopback(int64_t N, int32_t NB, int32_t P, int32_t Q, uint64_t seed,
                             int32_t device, hpl_ctx **out)
{
    if (!out) return HPL_ERR_ARG;
    const int nr = P * Q;
    if (check_args(N, NB, P, Q) != HPL_OK) return HPL_ERR_ARG;
    for (int r = 0; r < nr; ++r) out[r] = nullptr;
    if (nr > 1) {
        // Kernels of different ranks wait on each other on this one device:
        // they must be able to run at once.  Lazy module loading can
        // serialise a first launch behind running kernels, and too few
        // hardware queues put different ranks' streams in one FIFO; both are
        // fixed by the environment before the CUDA context exists.
        const char *ml = getenv("CUDA_MODULE_LOADING");
        const char *mc = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
        if (!ml || strcmp(ml, "EAGER") != 0 || !mc || atoi(mc) < 3 * nr) return HPL_ERR_STATE;
    }
    std::vector<hpl_ctx *> cs(nr, nullptr);
    hpl_status s = HPL_OK;
    if (cudaSetDevice(device) != cudaSuccess) return HPL_ERR_CUDA;
    for (int r = 0; r < nr && s == HPL_OK; ++r) {
        hpl_ctx *c = cs[r] = new hpl_ctx();
        c->N = N; c->NB = NB; c->P = P; c->Q = Q; c->seed = seed;
        c->rank = r; c->nranks = nr; c->myrow = r % P; c->mycol = r / P;
        c->device = device;
        c->dist = nr > 1;
        c->loop = true;
        s = alloc_ctx(c);
    }
    if (s == HPL_OK && nr > 1) {
        // the ranks share this device: they all grow, or none does
        const int want = panels_wanted(cs[0], nr);
        for (int r = 0; r < nr && s == HPL_OK; ++r) s = grow_panels(cs[r], want);
    }
    std::vector<PeerExports> ex(nr);
    for (int r = 0; r < nr && s == HPL_OK; ++r) ex[r] = exports_of(cs[r]);
    for (int r = 0; r < nr && s == HPL_OK; ++r) s = setup_peers(cs[r], ex);
    for (int r = 0; r < nr && s == HPL_OK; ++r) s = generate(cs[r]);
    for (int r = 0; r < nr; ++r) out[r] = cs[r];   // returned even on failure; caller frees
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

}  // extern "C"
