// Device ingestion of sampled configurations (SQD loop integration).
//
// Reference: ingest_samples (basis.py:251-313) filters sampled determinants
// by per-spin electron count, drops duplicates keeping FIRST-SEEN order,
// counts multiplicities (det_counts, used for the start vector in
// cli.py:117-128), and collects the unique alpha and beta halves in
// first-seen order (the product basis spans them).
//
// B200 formulation, all on the device: a filter + order-preserving
// compaction, a stable LSD radix sort of the kept samples by (alpha, beta)
// (beta pass, then a stable alpha pass), segment heads give each unique
// determinant's first sample (stability keeps ties in sample order) and its
// multiplicity; sorting the heads by first-sample index restores first-seen
// order.  The unique halves come from the same pattern on one key.  The first
// occurrence of an alpha (beta) string among the kept samples is always a new
// determinant, so this equals the reference's bookkeeping.
#include <algorithm>

#include "sbd_internal.cuh"

namespace {

constexpr int kScanBlock = 1024;
constexpr int kScanItems = 4;  // per thread
constexpr int kScanTile = kScanBlock * kScanItems;

// exclusive scan of int32 flags/counts, three kernels (tile scan, tile sums, add)
__global__ void scan_tiles(const int32_t *__restrict__ in, i64 n, int32_t *__restrict__ out,
                           int64_t *__restrict__ tile_sum) {
    __shared__ int32_t warp_tot[kScanBlock / 32];
    const i64 base = (i64)blockIdx.x * kScanTile + (i64)threadIdx.x * kScanItems;
    int32_t v[kScanItems], s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < n ? in[base + k] : 0;
        s += v[k];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    if (w == 0) {
        int32_t t = lane < kScanBlock / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        if (lane < kScanBlock / 32) warp_tot[lane] = t;
    }
    __syncthreads();
    int32_t run = inc - s + (w > 0 ? warp_tot[w - 1] : 0);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    if (threadIdx.x == kScanBlock - 1) tile_sum[blockIdx.x] = (int64_t)warp_tot[kScanBlock / 32 - 1];
}

__global__ void scan_tile_sums(int64_t *__restrict__ tile_sum, i64 ntiles, int64_t *__restrict__ total) {
    if (threadIdx.x != 0) return;
    int64_t run = 0;
    for (i64 t = 0; t < ntiles; ++t) {
        const int64_t v = tile_sum[t];
        tile_sum[t] = run;
        run += v;
    }
    *total = run;
}

__global__ void scan_add(int32_t *__restrict__ out, i64 n, const int64_t *__restrict__ tile_sum) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += (int32_t)tile_sum[i / kScanTile];
}

__global__ void filter_kernel(const u64 *__restrict__ a, const u64 *__restrict__ b, i64 n, int norb, int na, int nb,
                              int32_t *__restrict__ keep, int *__restrict__ bad) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const u64 hi = norb >= 64 ? 0 : ~(((u64)1 << norb) - 1);
    if ((a[i] & hi) || (b[i] & hi)) *bad = 1;
    keep[i] = (__popcll(a[i]) == na && __popcll(b[i]) == nb) ? 1 : 0;
}

__global__ void compact_kernel(const u64 *__restrict__ a, const u64 *__restrict__ b, const int32_t *__restrict__ keep,
                               const int32_t *__restrict__ pos, i64 n, u64 *__restrict__ ka, u64 *__restrict__ kb) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && keep[i]) {
        ka[pos[i]] = a[i];
        kb[pos[i]] = b[i];
    }
}

__global__ void gather_u64(const u64 *__restrict__ src, const int32_t *__restrict__ idx, i64 n, u64 *__restrict__ dst) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

__global__ void gather_i32(const int32_t *__restrict__ src, const int32_t *__restrict__ idx, i64 n,
                           int32_t *__restrict__ dst) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

// head flags of equal runs in sorted (key1[, key2]) order
__global__ void heads_kernel(const u64 *__restrict__ k1, const u64 *__restrict__ k2, i64 n, int32_t *__restrict__ head) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    head[i] = (i == 0 || k1[i] != k1[i - 1] || (k2 && k2[i] != k2[i - 1])) ? 1 : 0;
}

// per run: first sample index (the sample order of the run's head) and length
__global__ void runs_kernel(const int32_t *__restrict__ head, const int32_t *__restrict__ run_id,
                            const int32_t *__restrict__ order, i64 n, i64 nruns, u64 *__restrict__ first,
                            int32_t *__restrict__ start) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (head[i]) {
        first[run_id[i]] = (u64)order[i];
        start[run_id[i]] = (int32_t)i;
    }
    if (i == n - 1) start[nruns] = (int32_t)n;
}

__global__ void run_values(const int32_t *__restrict__ start, const int32_t *__restrict__ order_by_first, i64 nruns,
                           const u64 *__restrict__ key1, const u64 *__restrict__ key2, u64 *__restrict__ out1,
                           u64 *__restrict__ out2, int64_t *__restrict__ count) {
    const i64 u = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= nruns) return;
    const int32_t r = order_by_first[u];
    const int32_t s = start[r];
    out1[u] = key1[s];
    if (out2) out2[u] = key2[s];
    if (count) count[u] = start[r + 1] - s;
}

int scan_i32(sbd_ctx *ctx, const int32_t *in, i64 n, int32_t *out, int64_t *total_host) {
    cudaStream_t st = ctx->stream;
    const i64 ntiles = std::max<i64>(1, (n + kScanTile - 1) / kScanTile);
    DevBuf sums, tot;
    SBD_CUDA(ctx, sums.ensure(sizeof(int64_t) * (ntiles + 1)));
    SBD_CUDA(ctx, tot.ensure(sizeof(int64_t)));
    scan_tiles<<<(unsigned)ntiles, kScanBlock, 0, st>>>(in, n, out, sums.as<int64_t>());
    scan_tile_sums<<<1, 32, 0, st>>>(sums.as<int64_t>(), ntiles, tot.as<int64_t>());
    scan_add<<<grid_for(n, 256), 256, 0, st>>>(out, n, sums.as<int64_t>());
    SBD_LAUNCHED(ctx, "scan");
    SBD_CUDA(ctx, cudaMemcpyAsync(total_host, tot.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    return SBD_OK;
}

int bits_for(u64 v) {
    int b = 1;
    while (b < 64 && ((u64)1 << b) <= v) ++b;
    return b;
}

// unique values of k1 (k2) over `order`-sorted samples, in first-seen order.
// sorted1/sorted2: keys in sorted order; order: sample index of each sorted slot.
int unique_first_seen(sbd_ctx *ctx, const u64 *sorted1, const u64 *sorted2, const int32_t *order, i64 n,
                      DevBuf &out1, DevBuf &out2, DevBuf *count, i64 *nuniq) {
    cudaStream_t st = ctx->stream;
    DevBuf head, rid, first, start, sfirst, operm;
    SBD_CUDA(ctx, head.ensure(sizeof(int32_t) * (n + 1)));
    SBD_CUDA(ctx, rid.ensure(sizeof(int32_t) * (n + 1)));
    heads_kernel<<<grid_for(n, 256), 256, 0, st>>>(sorted1, sorted2, n, head.as<int32_t>());
    int64_t nr = 0;
    int rc = scan_i32(ctx, head.as<int32_t>(), n, rid.as<int32_t>(), &nr);
    if (rc) return rc;
    SBD_CUDA(ctx, first.ensure(sizeof(u64) * (nr + 1)));
    SBD_CUDA(ctx, start.ensure(sizeof(int32_t) * (nr + 1)));
    runs_kernel<<<grid_for(n, 256), 256, 0, st>>>(head.as<int32_t>(), rid.as<int32_t>(), order, n, nr,
                                                  first.as<u64>(), start.as<int32_t>());
    SBD_LAUNCHED(ctx, "runs");
    rc = sbd_radix_sort(ctx, first.as<u64>(), nr, bits_for((u64)n), sfirst, operm);
    if (rc) return rc;
    SBD_CUDA(ctx, out1.ensure(sizeof(u64) * (nr + 1)));
    if (sorted2) SBD_CUDA(ctx, out2.ensure(sizeof(u64) * (nr + 1)));
    if (count) SBD_CUDA(ctx, count->ensure(sizeof(int64_t) * (nr + 1)));
    run_values<<<grid_for(nr, 256), 256, 0, st>>>(start.as<int32_t>(), operm.as<int32_t>(), nr, sorted1, sorted2,
                                                  out1.as<u64>(), sorted2 ? out2.as<u64>() : nullptr,
                                                  count ? count->as<int64_t>() : nullptr);
    SBD_LAUNCHED(ctx, "run values");
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    *nuniq = nr;
    return SBD_OK;
}

__global__ void rank_of_run(const int32_t *__restrict__ order_by_first, i64 nruns, int32_t *__restrict__ rank) {
    const i64 u = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < nruns) rank[order_by_first[u]] = (int32_t)u;
}

// rid is the EXCLUSIVE scan of the head flags: the run of slot i is rid[i] + head[i] - 1
__global__ void index_of_sample(const int32_t *__restrict__ order, const int32_t *__restrict__ rid,
                                const int32_t *__restrict__ head, const int32_t *__restrict__ rank, i64 n,
                                int32_t *__restrict__ index) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) index[order[i]] = rank[rid[i] + head[i] - 1];
}

}  // namespace

// Unique values of keys[0..n) in first-seen order (uniq, *nuniq) and, per element, the position of its
// value in that list (index, device int32[n]) -- the explicit basis's string dedupe (sbd_set_dets).
int sbd_unique_first_seen_index(sbd_ctx *ctx, const u64 *keys, i64 n, int key_bits, DevBuf &uniq, i64 *nuniq,
                                int32_t *index) {
    cudaStream_t st = ctx->stream;
    *nuniq = 0;
    if (n == 0) return SBD_OK;
    DevBuf sorted, perm, head, rid, first, start, sfirst, operm, rank;
    int rc = sbd_radix_sort(ctx, keys, n, key_bits, sorted, perm);
    if (rc) return rc;
    SBD_CUDA(ctx, head.ensure(sizeof(int32_t) * (n + 1)));
    SBD_CUDA(ctx, rid.ensure(sizeof(int32_t) * (n + 1)));
    heads_kernel<<<grid_for(n, 256), 256, 0, st>>>(sorted.as<u64>(), nullptr, n, head.as<int32_t>());
    int64_t nr = 0;
    rc = scan_i32(ctx, head.as<int32_t>(), n, rid.as<int32_t>(), &nr);
    if (rc) return rc;
    SBD_CUDA(ctx, first.ensure(sizeof(u64) * (nr + 1)));
    SBD_CUDA(ctx, start.ensure(sizeof(int32_t) * (nr + 1)));
    runs_kernel<<<grid_for(n, 256), 256, 0, st>>>(head.as<int32_t>(), rid.as<int32_t>(), perm.as<int32_t>(), n, nr,
                                                  first.as<u64>(), start.as<int32_t>());
    SBD_LAUNCHED(ctx, "runs");
    rc = sbd_radix_sort(ctx, first.as<u64>(), nr, bits_for((u64)n), sfirst, operm);
    if (rc) return rc;
    SBD_CUDA(ctx, uniq.ensure(sizeof(u64) * (nr + 1)));
    SBD_CUDA(ctx, rank.ensure(sizeof(int32_t) * (nr + 1)));
    run_values<<<grid_for(nr, 256), 256, 0, st>>>(start.as<int32_t>(), operm.as<int32_t>(), nr, sorted.as<u64>(),
                                                  nullptr, uniq.as<u64>(), nullptr, nullptr);
    rank_of_run<<<grid_for(nr, 256), 256, 0, st>>>(operm.as<int32_t>(), nr, rank.as<int32_t>());
    index_of_sample<<<grid_for(n, 256), 256, 0, st>>>(perm.as<int32_t>(), rid.as<int32_t>(), head.as<int32_t>(),
                                                      rank.as<int32_t>(), n, index);
    SBD_LAUNCHED(ctx, "first-seen index");
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    *nuniq = nr;
    return SBD_OK;
}

extern "C" {

int sbd_ingest_samples(sbd_ctx *ctx, const uint64_t *alpha, const uint64_t *beta, int64_t n, int norb,
                       int n_alpha_elec, int n_beta_elec, int64_t *n_filtered, int64_t *n_unique_dets,
                       int64_t *n_unique_alpha, int64_t *n_unique_beta) {
    SBD_CHECK_CTX(ctx);
    if (n < 0 || (n > 0 && (!alpha || !beta))) return sbd_fail(ctx, SBD_EINVAL, "bad sample arrays");
    if (n >= (int64_t)INT32_MAX) return sbd_fail(ctx, SBD_EINVAL, "too many samples");
    if (norb < 1 || norb > 64) return sbd_fail(ctx, SBD_EINVAL, "norb must be in [1, 64]");
    cudaStream_t st = ctx->stream;
    IngestState &g = ctx->ingest;
    g.ready = false;
    g.n_det = g.n_alpha = g.n_beta = g.n_samples = g.n_kept = 0;
    DevBuf da, db, keep, pos, bad;
    SBD_CUDA(ctx, da.ensure(sizeof(u64) * (n + 1)));
    SBD_CUDA(ctx, db.ensure(sizeof(u64) * (n + 1)));
    SBD_CUDA(ctx, keep.ensure(sizeof(int32_t) * (n + 1)));
    SBD_CUDA(ctx, pos.ensure(sizeof(int32_t) * (n + 1)));
    SBD_CUDA(ctx, bad.ensure(sizeof(int)));
    if (n) {
        SBD_CUDA(ctx, cudaMemcpyAsync(da.p, alpha, sizeof(u64) * n, cudaMemcpyHostToDevice, st));
        SBD_CUDA(ctx, cudaMemcpyAsync(db.p, beta, sizeof(u64) * n, cudaMemcpyHostToDevice, st));
    }
    SBD_CUDA(ctx, cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    filter_kernel<<<grid_for(n, 256), 256, 0, st>>>(da.as<u64>(), db.as<u64>(), n, norb, n_alpha_elec, n_beta_elec,
                                                    keep.as<int32_t>(), bad.as<int>());
    SBD_LAUNCHED(ctx, "filter");
    int hbad = 0;
    SBD_CUDA(ctx, cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    int64_t nk = 0;
    int rc = scan_i32(ctx, keep.as<int32_t>(), n, pos.as<int32_t>(), &nk);
    if (rc) return rc;
    if (hbad) return sbd_fail(ctx, SBD_EINVAL, "sample has bits at or above norb");
    DevBuf ka, kb;
    SBD_CUDA(ctx, ka.ensure(sizeof(u64) * (nk + 1)));
    SBD_CUDA(ctx, kb.ensure(sizeof(u64) * (nk + 1)));
    compact_kernel<<<grid_for(n, 256), 256, 0, st>>>(da.as<u64>(), db.as<u64>(), keep.as<int32_t>(), pos.as<int32_t>(),
                                                     n, ka.as<u64>(), kb.as<u64>());
    SBD_LAUNCHED(ctx, "compact");
    // determinants: stable sort by beta, then by alpha
    DevBuf sb1, p1, a1, sa2, p2, order, bsorted;
    rc = sbd_radix_sort(ctx, kb.as<u64>(), nk, norb, sb1, p1);
    if (rc) return rc;
    SBD_CUDA(ctx, a1.ensure(sizeof(u64) * (nk + 1)));
    gather_u64<<<grid_for(nk, 256), 256, 0, st>>>(ka.as<u64>(), p1.as<int32_t>(), nk, a1.as<u64>());
    rc = sbd_radix_sort(ctx, a1.as<u64>(), nk, norb, sa2, p2);
    if (rc) return rc;
    SBD_CUDA(ctx, order.ensure(sizeof(int32_t) * (nk + 1)));
    SBD_CUDA(ctx, bsorted.ensure(sizeof(u64) * (nk + 1)));
    gather_i32<<<grid_for(nk, 256), 256, 0, st>>>(p1.as<int32_t>(), p2.as<int32_t>(), nk, order.as<int32_t>());
    gather_u64<<<grid_for(nk, 256), 256, 0, st>>>(kb.as<u64>(), order.as<int32_t>(), nk, bsorted.as<u64>());
    SBD_LAUNCHED(ctx, "gather");
    rc = unique_first_seen(ctx, sa2.as<u64>(), bsorted.as<u64>(), order.as<int32_t>(), nk, g.det_a, g.det_b,
                           &g.det_count, &g.n_det);
    if (rc) return rc;
    // unique halves
    DevBuf s1, pp;
    rc = sbd_radix_sort(ctx, ka.as<u64>(), nk, norb, s1, pp);
    if (rc) return rc;
    DevBuf dummy;
    rc = unique_first_seen(ctx, s1.as<u64>(), nullptr, pp.as<int32_t>(), nk, g.alpha, dummy, nullptr, &g.n_alpha);
    if (rc) return rc;
    rc = sbd_radix_sort(ctx, kb.as<u64>(), nk, norb, s1, pp);
    if (rc) return rc;
    rc = unique_first_seen(ctx, s1.as<u64>(), nullptr, pp.as<int32_t>(), nk, g.beta, dummy, nullptr, &g.n_beta);
    if (rc) return rc;
    g.n_samples = n;
    g.n_kept = nk;
    g.ready = true;
    if (n_filtered) *n_filtered = n - nk;
    if (n_unique_dets) *n_unique_dets = g.n_det;
    if (n_unique_alpha) *n_unique_alpha = g.n_alpha;
    if (n_unique_beta) *n_unique_beta = g.n_beta;
    return SBD_OK;
}

int sbd_ingest_export(sbd_ctx *ctx, uint64_t *det_alpha, uint64_t *det_beta, int64_t *det_count,
                      uint64_t *alpha_strings, uint64_t *beta_strings) {
    SBD_CHECK_CTX(ctx);
    IngestState &g = ctx->ingest;
    if (!g.ready) return sbd_fail(ctx, SBD_EINVAL, "no ingested samples (call sbd_ingest_samples)");
    cudaStream_t st = ctx->stream;
    auto down = [&](void *dst, const DevBuf &src, size_t bytes) -> cudaError_t {
        if (!dst || !bytes) return cudaSuccess;
        return cudaMemcpyAsync(dst, src.p, bytes, cudaMemcpyDeviceToHost, st);
    };
    SBD_CUDA(ctx, down(det_alpha, g.det_a, sizeof(u64) * g.n_det));
    SBD_CUDA(ctx, down(det_beta, g.det_b, sizeof(u64) * g.n_det));
    SBD_CUDA(ctx, down(det_count, g.det_count, sizeof(int64_t) * g.n_det));
    SBD_CUDA(ctx, down(alpha_strings, g.alpha, sizeof(u64) * g.n_alpha));
    SBD_CUDA(ctx, down(beta_strings, g.beta, sizeof(u64) * g.n_beta));
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    return SBD_OK;
}

}  // extern "C"
