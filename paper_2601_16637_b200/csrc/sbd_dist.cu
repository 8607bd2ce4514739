// Alpha-block partitioned sigma over GPUs, one process (context) per GPU, NCCL
// over NVLink/NVSwitch inside the library (reference DistributedApplier and
// its ring, distsim.py:130-316, 200-259).
//
// Partition (make_partition, distsim.py:63-77): rank r owns alpha rows
// [lo_r, hi_r) x all beta -- its x, sigma, diagonal and Davidson vectors.
// The beta-beta part of sigma needs only the owned rows; the alpha-alpha and
// alpha-beta (task 0) parts read the x rows the owned rows connect to, most
// of which live on other ranks.
//
// Exchange plan (sbd_dist_plan, collective).  x_work holds, in arrival order,
// segment 0 = the owned rows and segment s = the rows needed from peer
// (r - s) mod P, which arrive at ring step s (send to (r + s) mod P, receive
// from (r - s) mod P: the reference ring's neighbour pattern, with NVSwitch
// giving every pair full bandwidth).  Dense plans move whole blocks; sparse
// plans move only the rows some owned row references, packed
// by the sender.  The owned rows' alpha connections are remapped to x_work
// rows and sorted by them, so the connections into any run of segments are
// one contiguous range per row.
//
// Schedule of one sbd_sigma_dist (compute stream st, exchange stream cs):
//   cs:  wait(x ready) | x_own -> segment 0 | group 1 steps | group 2 steps | ...
//   st:  beta side (owned rows) | alpha pass over segment 0 + diag + (B X^T)^T
//        | wait(group 1) | alpha pass over group 1's segments (y +=) | ...
//        | task 0 (y +=, all segments)
// so the transfers overlap the beta side and the alpha work of the blocks
// that already landed; only the last group's transfer can be exposed.
// Profiling mode records per-step compute / transfer / exposed times
// (the reference's StepStat / overlap_stats, distsim.py:81-88,340-367).
#include <dlfcn.h>
#include <unistd.h>
#include <nccl.h>  // types only: the symbols are resolved at run time (dlopen)

#include <algorithm>
#include <cstring>
#include <type_traits>

#include "sbd_internal.cuh"

namespace {

// ---- NCCL, loaded on first use: the library does not link it, so a process
// that never goes multi-GPU never needs it, and under PyTorch the already
// loaded libnccl.so.2 (same soname) is reused.
struct Nccl {
    bool tried = false, ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*GetVersion)(int *) = nullptr;
};

Nccl &nccl() {
    static Nccl n;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (n.tried) return n;
    n.tried = true;
    const char *env = getenv("SBD_NCCL_LIB");
    const char *names[] = {env, "libnccl.so.2", "libnccl.so"};
    void *h = nullptr;
    for (const char *nm : names)
        if (nm && *nm && (h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
        n.err = std::string("cannot load libnccl.so.2: ") + dlerror();
        return n;
    }
    bool all = true;
    auto sym = [&](auto &fn, const char *name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        if (!fn) all = false;
    };
    sym(n.GetUniqueId, "ncclGetUniqueId");
    sym(n.CommInitRank, "ncclCommInitRank");
    sym(n.CommDestroy, "ncclCommDestroy");
    sym(n.CommAbort, "ncclCommAbort");
    sym(n.CommGetAsyncError, "ncclCommGetAsyncError");
    sym(n.GetErrorString, "ncclGetErrorString");
    sym(n.AllReduce, "ncclAllReduce");
    sym(n.AllGather, "ncclAllGather");
    sym(n.Send, "ncclSend");
    sym(n.Recv, "ncclRecv");
    sym(n.GroupStart, "ncclGroupStart");
    sym(n.GroupEnd, "ncclGroupEnd");
    sym(n.GetVersion, "ncclGetVersion");
    if (!all) {
        n.err = "libnccl.so.2 lacks a required symbol";
        return n;
    }
    n.ok = true;
    return n;
}

int nccl_fail(sbd_ctx *ctx, ncclResult_t r, const char *where) {
    const Nccl &n = nccl();
    std::string m = std::string(where) + ": NCCL error " + std::to_string((int)r);
    if (n.GetErrorString) m += std::string(" (") + n.GetErrorString(r) + ")";
    return sbd_fail(ctx, SBD_ECUDA, m);
}

#define SBD_NCCL(ctx, call)                                      \
    do {                                                         \
        ncclResult_t _r = (call);                                \
        if (_r != ncclSuccess) return nccl_fail((ctx), _r, #call); \
    } while (0)

inline ncclComm_t comm_of(const sbd_ctx *ctx) { return reinterpret_cast<ncclComm_t>(ctx->dist.comm); }

int groups_of(const DistState &d) { return (d.nranks - 1 + d.group_steps - 1) / d.group_steps; }
int group_first(const DistState &d, int g) { return 1 + g * d.group_steps; }
int group_last(const DistState &d, int g) { return std::min(d.nranks - 1, (g + 1) * d.group_steps); }

// dst[i, :] = src[rows[i], :]  (sparse exchange: pack the rows a peer asked for)
__global__ void pack_rows_kernel(const double *__restrict__ src, const int32_t *__restrict__ rows, i64 cnt, i64 nb,
                                 double *__restrict__ dst) {
    for (i64 i = blockIdx.x; i < cnt; i += gridDim.x) {
        const double *s = src + (i64)rows[i] * nb;
        double *d = dst + i * nb;
        for (i64 c = threadIdx.x; c < nb; c += blockDim.x) d[c] = __ldcs(s + c);
    }
}

int ensure_dist_events(sbd_ctx *ctx) {
    DistState &d = ctx->dist;
    const size_t need = (size_t)groups_of(d) + 1;
    while (d.ev.size() < need) {
        cudaEvent_t e;
        SBD_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        d.ev.push_back(e);
    }
    // timing: t_start, t_local, per group (pre, post, done), c_start, per group c_g
    const size_t tneed = 3 + 4 * (size_t)groups_of(d);
    while (d.tev.size() < tneed) {
        cudaEvent_t e;
        SBD_CUDA(ctx, cudaEventCreate(&e));
        d.tev.push_back(e);
    }
    return SBD_OK;
}

// Accumulate the timing events of the last profiled sigma.
int harvest(sbd_ctx *ctx) {
    DistState &d = ctx->dist;
    if (!d.tev_pending) return SBD_OK;
    d.tev_pending = false;
    const int G = groups_of(d);
    cudaEvent_t *t = d.tev.data();
    // layout: 0 t_start, 1 t_local, 2 c_start, then per group g: 3+4g pre, 4+4g post, 5+4g done, 6+4g c_g
    SBD_CUDA(ctx, cudaEventSynchronize(t[5 + 4 * (G - 1)]));
    auto el = [&](cudaEvent_t a, cudaEvent_t b) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        return (double)ms;
    };
    if (d.compute_ms.size() < (size_t)G + 1) {
        d.compute_ms.assign(G + 1, 0.0);
        d.transfer_ms.assign(G + 1, 0.0);
        d.exposed_ms.assign(G + 1, 0.0);
    }
    d.compute_ms[0] += el(t[0], t[1]);
    for (int g = 0; g < G; ++g) {
        d.exposed_ms[g + 1] += el(t[3 + 4 * g], t[4 + 4 * g]);
        d.compute_ms[g + 1] += el(t[4 + 4 * g], t[5 + 4 * g]);
        d.transfer_ms[g + 1] += el(g ? t[6 + 4 * (g - 1)] : t[2], t[6 + 4 * g]);
    }
    d.total_ms += el(t[0], t[5 + 4 * (G - 1)]);
    d.n_sigma++;
    return SBD_OK;
}

int allreduce_dev(sbd_ctx *ctx, void *buf, size_t n, ncclDataType_t ty, ncclRedOp_t op, cudaStream_t st) {
    if (!ctx->dist.on || ctx->dist.nranks == 1 || n == 0) return SBD_OK;
    SBD_NCCL(ctx, nccl().AllReduce(buf, buf, n, ty, op, comm_of(ctx), st));
    return SBD_OK;
}

int check_async(sbd_ctx *ctx) {
    if (!ctx->dist.on || !ctx->dist.comm) return SBD_OK;
    ncclResult_t ae = ncclSuccess;
    SBD_NCCL(ctx, nccl().CommGetAsyncError(comm_of(ctx), &ae));
    if (ae != ncclSuccess && ae != ncclInProgress) return nccl_fail(ctx, ae, "NCCL asynchronous error");
    return SBD_OK;
}

// The collective exchange plan; every rank calls it with the same arguments.
int plan(sbd_ctx *ctx, int exchange, double threshold, int group_steps) {
    DistState &d = ctx->dist;
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    const int P = d.nranks, r = d.rank;
    const i64 lo = ctx->own_lo(), hi = ctx->own_hi(), rows = hi - lo, na = A.n, nb = B.n;
    cudaStream_t st = ctx->stream;
    d.planned = false;
    d.group_steps = std::max(1, std::min(group_steps, std::max(P - 1, 1)));
    // the owned rows' connections and task-0 singles
    std::vector<int64_t> off(rows + 1), soff(2);
    SBD_CUDA(ctx, cudaMemcpyAsync(off.data(), A.conn_off.as<int64_t>() + lo, sizeof(int64_t) * (rows + 1),
                                  cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaMemcpyAsync(&soff[0], A.s_off.as<int64_t>() + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaMemcpyAsync(&soff[1], A.s_off.as<int64_t>() + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    const i64 nconn = off[rows] - off[0];
    std::vector<Conn> conn(nconn);
    if (nconn)
        SBD_CUDA(ctx, cudaMemcpy(conn.data(), A.conn.as<Conn>() + off[0], sizeof(Conn) * nconn, cudaMemcpyDeviceToHost));
    std::vector<SConn> sconn(A.ns);
    if (A.ns) SBD_CUDA(ctx, cudaMemcpy(sconn.data(), A.sconn.p, sizeof(SConn) * A.ns, cudaMemcpyDeviceToHost));

    // referenced remote rows (task-0 targets are singles, a subset of the connections)
    std::vector<char> ref(na, 0);
    for (const Conn &c : conn) ref[c.tgt] = 1;
    std::vector<std::vector<int32_t>> need(P);
    i64 n_need = 0;
    for (int q = 0; q < P; ++q) {
        if (q == r) continue;
        for (i64 ja = d.blk[q]; ja < d.blk[q + 1]; ++ja)
            if (ref[ja]) need[q].push_back((int32_t)ja);
        n_need += (i64)need[q].size();
    }
    // the dense/sparse decision must agree on every rank: the largest needed fraction decides
    DevBuf tmp;
    SBD_CUDA(ctx, tmp.ensure(sizeof(int64_t) * (size_t)P * P + 64));
    double frac = na > rows ? (double)n_need / (double)(na - rows) : 0.0;
    SBD_CUDA(ctx, cudaMemcpyAsync(tmp.p, &frac, sizeof(double), cudaMemcpyHostToDevice, st));
    if (int rc = allreduce_dev(ctx, tmp.p, 1, ncclFloat64, ncclMax, st)) return rc;
    SBD_CUDA(ctx, cudaMemcpyAsync(&frac, tmp.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    d.needed_fraction = frac;
    d.sparse = exchange == 2 || (exchange == 0 && frac <= threshold);
    if (!d.sparse)
        for (int q = 0; q < P; ++q) {
            need[q].clear();
            if (q != r)
                for (i64 ja = d.blk[q]; ja < d.blk[q + 1]; ++ja) need[q].push_back((int32_t)ja);
        }

    // step s: receive need[(r - s) mod P] from that peer, send what (r + s) mod P needs from me
    d.recv_cnt.assign(P, 0);
    d.send_cnt.assign(P, 0);
    d.send_off.assign(P + 1, 0);
    for (int s = 1; s < P; ++s) d.recv_cnt[s] = (i64)need[(r - s + P) % P].size();
    std::vector<int32_t> send_rows;
    if (!d.sparse) {
        for (int s = 1; s < P; ++s) d.send_cnt[s] = rows;
    } else {
        // counts matrix cnt[p][q] = rows p needs from q, then the request lists themselves
        std::vector<int64_t> mine(P, 0), all((size_t)P * P, 0);
        for (int q = 0; q < P; ++q) mine[q] = (int64_t)need[q].size();
        DevBuf dm;
        SBD_CUDA(ctx, dm.ensure(sizeof(int64_t) * P));
        SBD_CUDA(ctx, cudaMemcpyAsync(dm.p, mine.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, st));
        SBD_NCCL(ctx, nccl().AllGather(dm.p, tmp.p, P, ncclInt64, comm_of(ctx), st));
        SBD_CUDA(ctx, cudaMemcpyAsync(all.data(), tmp.p, sizeof(int64_t) * P * P, cudaMemcpyDeviceToHost, st));
        SBD_CUDA(ctx, cudaStreamSynchronize(st));
        std::vector<i64> in_off(P + 1, 0), out_off(P + 1, 0);
        for (int p = 0; p < P; ++p) {
            in_off[p + 1] = in_off[p] + (p == r ? 0 : all[(size_t)p * P + r]);  // rows p asks of me
            out_off[p + 1] = out_off[p] + (i64)need[p].size();                  // rows I ask of p
        }
        std::vector<int32_t> out_lists(out_off[P]);
        for (int p = 0; p < P; ++p) std::copy(need[p].begin(), need[p].end(), out_lists.begin() + out_off[p]);
        DevBuf din, dout;
        SBD_CUDA(ctx, din.ensure(sizeof(int32_t) * (in_off[P] + 1)));
        SBD_CUDA(ctx, dout.ensure(sizeof(int32_t) * (out_off[P] + 1)));
        if (out_off[P])
            SBD_CUDA(ctx, cudaMemcpyAsync(dout.p, out_lists.data(), sizeof(int32_t) * out_off[P], cudaMemcpyHostToDevice, st));
        SBD_NCCL(ctx, nccl().GroupStart());
        for (int p = 0; p < P; ++p) {
            if (p == r) continue;
            if (out_off[p + 1] > out_off[p])
                SBD_NCCL(ctx, nccl().Send(dout.as<int32_t>() + out_off[p], out_off[p + 1] - out_off[p], ncclInt32, p,
                                          comm_of(ctx), st));
            if (in_off[p + 1] > in_off[p])
                SBD_NCCL(ctx, nccl().Recv(din.as<int32_t>() + in_off[p], in_off[p + 1] - in_off[p], ncclInt32, p,
                                          comm_of(ctx), st));
        }
        SBD_NCCL(ctx, nccl().GroupEnd());
        std::vector<int32_t> in_lists(in_off[P]);
        if (in_off[P])
            SBD_CUDA(ctx, cudaMemcpyAsync(in_lists.data(), din.p, sizeof(int32_t) * in_off[P], cudaMemcpyDeviceToHost, st));
        SBD_CUDA(ctx, cudaStreamSynchronize(st));
        for (int s = 1; s < P; ++s) {
            const int p = (r + s) % P;
            d.send_cnt[s] = in_off[p + 1] - in_off[p];
            d.send_off[s] = (i64)send_rows.size();
            for (i64 i = in_off[p]; i < in_off[p + 1]; ++i) send_rows.push_back((int32_t)(in_lists[i] - lo));
        }
        d.send_off[P] = (i64)send_rows.size();
    }

    // x_work layout and the remap of global alpha rows to x_work rows
    d.seg_start.assign(P + 1, 0);
    d.seg_start[1] = rows;
    for (int s = 1; s < P; ++s) d.seg_start[s + 1] = d.seg_start[s] + d.recv_cnt[s];
    std::vector<int32_t> map(na, -1);
    for (i64 ja = lo; ja < hi; ++ja) map[ja] = (int32_t)(ja - lo);
    for (int s = 1; s < P; ++s) {
        const std::vector<int32_t> &lst = need[(r - s + P) % P];
        for (size_t i = 0; i < lst.size(); ++i) map[lst[i]] = (int32_t)(d.seg_start[s] + (i64)i);
    }
    // remap + sort each owned row's connections by x_work row; segment offsets per row
    std::vector<int64_t> seg_off((size_t)rows * (P + 1));
    for (i64 i = 0; i < rows; ++i) {
        Conn *b = conn.data() + (off[i] - off[0]), *e = conn.data() + (off[i + 1] - off[0]);
        for (Conn *c = b; c < e; ++c) {
            if (map[c->tgt] < 0) return sbd_fail(ctx, SBD_ECUDA, "dist plan: unmapped alpha target");
            c->tgt = map[c->tgt];
        }
        std::sort(b, e, [](const Conn &x, const Conn &y) { return x.tgt < y.tgt; });
        Conn *c = b;
        for (int s = 0; s <= P; ++s) {
            const i64 bound = s < P ? d.seg_start[s] : INT64_MAX;
            while (c < e && (i64)c->tgt < bound) ++c;
            // seg_off[i][s] = first connection at or beyond segment s
            seg_off[(size_t)i * (P + 1) + s] = (s < P ? (i64)(c - conn.data()) : (i64)(e - conn.data()));
        }
    }
    for (i64 e = soff[0]; e < soff[1]; ++e) sconn[e].tgt = map[sconn[e].tgt];

    SBD_CUDA(ctx, d.conn.ensure(sizeof(Conn) * (nconn + 1)));
    SBD_CUDA(ctx, d.seg_off.ensure(sizeof(int64_t) * seg_off.size() + 8));
    SBD_CUDA(ctx, d.sconn.ensure(sizeof(SConn) * (A.ns + 1)));
    if (nconn) SBD_CUDA(ctx, cudaMemcpy(d.conn.p, conn.data(), sizeof(Conn) * nconn, cudaMemcpyHostToDevice));
    SBD_CUDA(ctx, cudaMemcpy(d.seg_off.p, seg_off.data(), sizeof(int64_t) * seg_off.size(), cudaMemcpyHostToDevice));
    if (A.ns) SBD_CUDA(ctx, cudaMemcpy(d.sconn.p, sconn.data(), sizeof(SConn) * A.ns, cudaMemcpyHostToDevice));
    SBD_CUDA(ctx, d.xw.ensure(sizeof(double) * ((size_t)d.seg_start[P] * nb + 2)));
    if (d.sparse) {
        SBD_CUDA(ctx, d.send_rows.ensure(sizeof(int32_t) * (send_rows.size() + 1)));
        if (!send_rows.empty())
            SBD_CUDA(ctx, cudaMemcpy(d.send_rows.p, send_rows.data(), sizeof(int32_t) * send_rows.size(),
                                     cudaMemcpyHostToDevice));
        SBD_CUDA(ctx, d.send_buf.ensure(sizeof(double) * ((size_t)send_rows.size() * nb + 2)));
    }
    if (int rc = ensure_dist_events(ctx)) return rc;
    d.planned = true;
    return SBD_OK;
}

}  // namespace

void sbd_dist_release(sbd_ctx *ctx) {
    DistState &d = ctx->dist;
    if (d.cs) {
        cudaStreamSynchronize(d.cs);
        cudaStreamDestroy(d.cs);
        d.cs = nullptr;
    }
    for (cudaEvent_t e : d.ev) cudaEventDestroy(e);
    for (cudaEvent_t e : d.tev) cudaEventDestroy(e);
    d.ev.clear();
    d.tev.clear();
    if (d.comm) {
        nccl().CommDestroy(comm_of(ctx));
        d.comm = nullptr;
    }
    d.on = false;
    d.planned = false;
}

// Internal (sbd_solver.cu): all-reduce n doubles on the context's stream; no-op on one rank.
int sbd_dist_allreduce_internal(sbd_ctx *ctx, double *buf, i64 n, int op) {
    const ncclRedOp_t o = op == 1 ? ncclMax : (op == 2 ? ncclMin : ncclSum);
    return allreduce_dev(ctx, buf, (size_t)n, ncclFloat64, o, ctx->stream);
}
int sbd_dist_check_internal(sbd_ctx *ctx) { return check_async(ctx); }

extern "C" {

int sbd_nccl_unique_id(char *id_out) {
    if (!id_out) return sbd_fail(nullptr, SBD_EINVAL, "sbd_nccl_unique_id: null output");
    Nccl &n = nccl();
    if (!n.ok) return sbd_fail(nullptr, SBD_ECUDA, n.err);
    ncclUniqueId id;
    ncclResult_t r = n.GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(nullptr, r, "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return SBD_OK;
}

int sbd_dist_init(sbd_ctx *ctx, int rank, int nranks, const char *id, const int64_t *alpha_edges) {
    SBD_CHECK_CTX(ctx);
    if (ctx->explicit_mode) return sbd_fail(ctx, SBD_EINVAL, "distributed application requires a product-mode basis");
    if (!ctx->sec[0].present) return sbd_fail(ctx, SBD_EINVAL, "set the alpha strings before sbd_dist_init");
    const i64 na = ctx->sec[0].n;
    if (nranks < 1) return sbd_fail(ctx, SBD_EINVAL, "need at least one worker, got " + std::to_string(nranks));
    if (nranks > na)
        return sbd_fail(ctx, SBD_EINVAL,
                        "cannot split " + std::to_string(na) + " alpha strings over " + std::to_string(nranks) + " workers");
    if (rank < 0 || rank >= nranks) return sbd_fail(ctx, SBD_EINVAL, "rank out of range");
    if (nranks > 1 && !id) return sbd_fail(ctx, SBD_EINVAL, "sbd_dist_init: null NCCL unique id");
    sbd_dist_release(ctx);
    DistState &d = ctx->dist;
    d.rank = rank;
    d.nranks = nranks;
    d.blk.assign(nranks + 1, 0);
    if (alpha_edges) {  // a caller's Partition: contiguous, non-empty blocks covering all rows
        for (int w = 0; w <= nranks; ++w) d.blk[w] = alpha_edges[w];
        bool ok = d.blk[0] == 0 && d.blk[nranks] == na;
        for (int w = 0; w < nranks; ++w) ok = ok && d.blk[w] < d.blk[w + 1];
        if (!ok) return sbd_fail(ctx, SBD_EINVAL, "alpha_edges must run 0 = e0 < e1 < ... < e_P = n_alpha");
    } else {  // make_partition (distsim.py:63-77): the first `rem` blocks one row longer
        const i64 base = na / nranks, rem = na % nranks;
        for (int w = 0; w < nranks; ++w) d.blk[w + 1] = d.blk[w] + base + (w < rem ? 1 : 0);
    }
    if (nranks > 1) {
        Nccl &n = nccl();
        if (!n.ok) return sbd_fail(ctx, SBD_ECUDA, n.err);
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
        ncclComm_t comm = nullptr;
        // NCCL announces its version on stdout during the first init; a library must not write to
        // the caller's stdout (the CLI's JSON report goes there), so it goes to stderr instead
        fflush(stdout);
        const int saved = dup(1);
        if (saved >= 0) dup2(2, 1);
        const ncclResult_t r = n.CommInitRank(&comm, nranks, uid, rank);
        fflush(stdout);
        if (saved >= 0) {
            dup2(saved, 1);
            close(saved);
        }
        if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclCommInitRank");
        d.comm = comm;
        SBD_CUDA(ctx, cudaStreamCreateWithFlags(&d.cs, cudaStreamNonBlocking));
    }
    d.on = true;
    d.planned = false;
    d.n_sigma = 0;
    ctx->row_lo = d.blk[rank];
    ctx->row_hi = d.blk[rank + 1];
    ctx->diag_valid = false;
    return SBD_OK;
}

int sbd_dist_plan(sbd_ctx *ctx, int exchange, double sparse_threshold, int group_steps) {
    SBD_CHECK_CTX(ctx);
    if (!ctx->dist.on) return sbd_fail(ctx, SBD_EINVAL, "sbd_dist_plan: call sbd_dist_init first");
    if (exchange < 0 || exchange > 2) return sbd_fail(ctx, SBD_EINVAL, "exchange must be 0 (auto), 1 (dense) or 2 (sparse)");
    if (group_steps < 1) return sbd_fail(ctx, SBD_EINVAL, "group_steps must be >= 1");
    if (int rc = sbd_require_sigma_ready(ctx)) return rc;
    if (ctx->dist.nranks == 1) {
        ctx->dist.planned = true;
        return SBD_OK;
    }
    return plan(ctx, exchange, sparse_threshold, group_steps);
}

int sbd_sigma_dist(sbd_ctx *ctx, const double *x_own, double *y_own) {
    SBD_CHECK_CTX(ctx);
    SbdRange range("sbd/sigma_dist");
    DistState &d = ctx->dist;
    if (!d.on) return sbd_fail(ctx, SBD_EINVAL, "sbd_sigma_dist: call sbd_dist_init first");
    if (!x_own || !y_own) return sbd_fail(ctx, SBD_EINVAL, "null vector");
    if (int rc = sbd_require_sigma_ready(ctx)) return rc;
    if (d.nranks == 1) return sbd_sigma(ctx, x_own, y_own);
    if (!d.planned)
        if (int rc = plan(ctx, 0, 0.6, 2)) return rc;
    if (int rc = harvest(ctx)) return rc;
    const int P = d.nranks, r = d.rank, G = groups_of(d);
    const i64 nb = ctx->sec[1].n, rows = ctx->own_rows();
    cudaStream_t st = ctx->stream, cs = d.cs;
    double *xw = d.xw.as<double>();
    const bool prof = d.profile;
    cudaEvent_t *t = d.tev.data();
    SBD_CUDA(ctx, cudaEventRecord(d.ev[0], st));  // x_own ready, earlier users of x_work done
    if (prof) SBD_CUDA(ctx, cudaEventRecord(t[0], st));
    SBD_CUDA(ctx, cudaStreamWaitEvent(cs, d.ev[0], 0));
    if (prof) SBD_CUDA(ctx, cudaEventRecord(t[2], cs));
    // ---- exchange stream
    SBD_CUDA(ctx, cudaMemcpyAsync(xw, x_own, sizeof(double) * rows * nb, cudaMemcpyDeviceToDevice, cs));
    for (int g = 0; g < G; ++g) {
        const int s0 = group_first(d, g), s1 = group_last(d, g);
        if (d.sparse)
            for (int s = s0; s <= s1; ++s)
                if (d.send_cnt[s]) {
                    const unsigned blocks = (unsigned)std::min<i64>(d.send_cnt[s], 8 * (i64)ctx->num_sms);
                    pack_rows_kernel<<<blocks, 256, 0, cs>>>(x_own, d.send_rows.as<int32_t>() + d.send_off[s],
                                                             d.send_cnt[s], nb, d.send_buf.as<double>() + d.send_off[s] * nb);
                    SBD_LAUNCHED(ctx, "pack_rows_kernel");
                }
        SBD_NCCL(ctx, nccl().GroupStart());
        for (int s = s0; s <= s1; ++s) {
            const int to = (r + s) % P, from = (r - s + P) % P;
            if (d.send_cnt[s]) {
                const double *src = d.sparse ? d.send_buf.as<double>() + d.send_off[s] * nb : x_own;
                SBD_NCCL(ctx, nccl().Send(src, (size_t)(d.send_cnt[s] * nb), ncclFloat64, to, comm_of(ctx), cs));
            }
            if (d.recv_cnt[s])
                SBD_NCCL(ctx, nccl().Recv(xw + d.seg_start[s] * nb, (size_t)(d.recv_cnt[s] * nb), ncclFloat64, from,
                                          comm_of(ctx), cs));
        }
        SBD_NCCL(ctx, nccl().GroupEnd());
        SBD_CUDA(ctx, cudaEventRecord(d.ev[1 + g], cs));
        if (prof) SBD_CUDA(ctx, cudaEventRecord(t[6 + 4 * g], cs));
    }
    // ---- compute stream: owned-row work first, then each group as it lands
    if (int rc = sbd_beta_side(ctx, x_own)) return rc;
    const Conn *conn = d.conn.as<Conn>();
    const int64_t *so = d.seg_off.as<int64_t>();
    // segment 0 rows are x_own's rows: this pass does not wait for the exchange stream
    if (int rc = sbd_alpha_pass(ctx, x_own, y_own, conn, so, P + 1, 0, 1, 0, true, false)) return rc;
    if (prof) SBD_CUDA(ctx, cudaEventRecord(t[1], st));
    for (int g = 0; g < G; ++g) {
        if (prof) SBD_CUDA(ctx, cudaEventRecord(t[3 + 4 * g], st));
        SBD_CUDA(ctx, cudaStreamWaitEvent(st, d.ev[1 + g], 0));
        if (prof) SBD_CUDA(ctx, cudaEventRecord(t[4 + 4 * g], st));
        if (int rc = sbd_alpha_pass(ctx, xw, y_own, conn, so, P + 1, group_first(d, g), group_last(d, g) + 1, 0, false,
                                    true))
            return rc;
        if (g == G - 1)
            if (int rc = sbd_cross_add(ctx, xw, y_own, d.sconn.as<SConn>())) return rc;
        if (prof) SBD_CUDA(ctx, cudaEventRecord(t[5 + 4 * g], st));
    }
    d.tev_pending = prof;
    return SBD_OK;
}

int sbd_dist_allreduce(sbd_ctx *ctx, double *buf_dev, int64_t n, int op) {
    SBD_CHECK_CTX(ctx);
    if (!ctx->dist.on) return sbd_fail(ctx, SBD_EINVAL, "sbd_dist_allreduce: call sbd_dist_init first");
    if (op < 0 || op > 2) return sbd_fail(ctx, SBD_EINVAL, "op must be 0 (sum), 1 (max) or 2 (min)");
    if (n < 0 || (n > 0 && !buf_dev)) return sbd_fail(ctx, SBD_EINVAL, "bad buffer");
    return sbd_dist_allreduce_internal(ctx, buf_dev, n, op);
}

int sbd_dist_check(sbd_ctx *ctx) {
    SBD_CHECK_CTX(ctx);
    return check_async(ctx);
}

int sbd_dist_info(sbd_ctx *ctx, int *rank, int *nranks, int64_t *alpha_lo, int64_t *alpha_hi, int *sparse,
                  double *needed_fraction, int64_t *recv_rows, int64_t *send_rows, int *n_groups) {
    SBD_CHECK_CTX(ctx);
    const DistState &d = ctx->dist;
    if (!d.on) return sbd_fail(ctx, SBD_EINVAL, "sbd_dist_info: call sbd_dist_init first");
    if (rank) *rank = d.rank;
    if (nranks) *nranks = d.nranks;
    if (alpha_lo) *alpha_lo = ctx->own_lo();
    if (alpha_hi) *alpha_hi = ctx->own_hi();
    i64 rr = 0, sr = 0;
    if (d.planned && d.nranks > 1)
        for (int s = 1; s < d.nranks; ++s) rr += d.recv_cnt[s], sr += d.send_cnt[s];
    if (sparse) *sparse = d.planned ? d.sparse : -1;
    if (needed_fraction) *needed_fraction = d.needed_fraction;
    if (recv_rows) *recv_rows = rr;
    if (send_rows) *send_rows = sr;
    if (n_groups) *n_groups = d.nranks > 1 ? groups_of(d) : 0;
    return SBD_OK;
}

int sbd_dist_set_profiling(sbd_ctx *ctx, int on) {
    SBD_CHECK_CTX(ctx);
    DistState &d = ctx->dist;
    if (int rc = harvest(ctx)) return rc;
    d.profile = on != 0;
    d.n_sigma = 0;
    d.total_ms = 0.0;
    d.compute_ms.clear();
    d.transfer_ms.clear();
    d.exposed_ms.clear();
    return SBD_OK;
}

int sbd_dist_stats(sbd_ctx *ctx, int64_t *n_sigma, int *n_steps, double *compute_ms, double *transfer_ms,
                   double *exposed_ms, double *total_ms) {
    SBD_CHECK_CTX(ctx);
    DistState &d = ctx->dist;
    if (int rc = harvest(ctx)) return rc;
    if (int rc = check_async(ctx)) return rc;
    const int ns = (int)d.compute_ms.size();
    if (n_sigma) *n_sigma = d.n_sigma;
    if (n_steps) *n_steps = ns;
    for (int i = 0; i < ns; ++i) {
        if (compute_ms) compute_ms[i] = d.compute_ms[i];
        if (transfer_ms) transfer_ms[i] = d.transfer_ms[i];
        if (exposed_ms) exposed_ms[i] = d.exposed_ms[i];
    }
    if (total_ms) *total_ms = d.total_ms;
    return SBD_OK;
}

}  // extern "C"
