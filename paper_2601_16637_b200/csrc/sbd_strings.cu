// Configuration processing: device LSD radix sort + uniqueness check of one
// spin sector's strings.
//
// Reference: the sector's string list is caller-ordered (basis.py:138-160,
// 278-297) and build_excitation_table indexes it through a dict
// (basis.py:364-366), rejecting duplicates.  Here the device sorts the 64-bit
// masks once (keys = masks, values = caller index) so that excitation
// generation can find targets by binary search; perm maps a sorted position
// back to the caller index, so every table keeps caller-order indices.
//
// Sort: 8-bit LSD digits, only ceil(norb/8) passes (bits >= norb are zero).
// Per pass: tile histogram -> digit-major exclusive scan -> stable scatter
// (warp match_any ranking + per-warp digit prefix), tiles of 1024 keys.
// Keys are one word (u64) or two (U128, norb <= 128: the digit passes walk
// the low word, then the high one).
#include <algorithm>

#include "sbd_internal.cuh"
#include "sbd_words.cuh"

namespace {

constexpr int kTile = 1024;  // keys per block == threads per block
constexpr int kWarps = kTile / 32;

template <class W>
__global__ void radix_hist(const W *__restrict__ keys, i64 n, int shift, int *__restrict__ hist, int nblocks) {
    __shared__ int h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    i64 i = (i64)blockIdx.x * kTile + threadIdx.x;
    if (i < n) atomicAdd(&h[words::digit(keys[i], shift)], 1);
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[d * nblocks + blockIdx.x] = h[d];
}

// single-block exclusive scan of m ints (m = 256 * nblocks, small)
__global__ void exclusive_scan_small(int *__restrict__ a, int m) {
    __shared__ int part[1024];
    int t = threadIdx.x, nt = blockDim.x;
    int per = (m + nt - 1) / nt;
    int lo = t * per, hi = min(m, lo + per);
    int s = 0;
    for (int i = lo; i < hi; ++i) s += a[i];
    part[t] = s;
    __syncthreads();
    if (t == 0) {
        int run = 0;
        for (int i = 0; i < nt; ++i) {
            int v = part[i];
            part[i] = run;
            run += v;
        }
    }
    __syncthreads();
    int run = part[t];
    for (int i = lo; i < hi; ++i) {
        int v = a[i];
        a[i] = run;
        run += v;
    }
}

template <class W>
__global__ void radix_scatter(const W *__restrict__ kin, const int32_t *__restrict__ vin, W *__restrict__ kout,
                              int32_t *__restrict__ vout, i64 n, int shift, const int *__restrict__ offs,
                              int nblocks) {
    __shared__ int cnt[kWarps][256];
    int t = threadIdx.x, w = t >> 5, lane = t & 31;
    for (int i = t; i < kWarps * 256; i += kTile) (&cnt[0][0])[i] = 0;
    __syncthreads();
    i64 i = (i64)blockIdx.x * kTile + t;
    bool valid = i < n;
    W key{};
    if (valid) key = kin[i];
    int d = valid ? words::digit(key, shift) : 256 + lane;  // invalid lanes never match valid ones
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int rank = __popc(peers & ((1u << lane) - 1));
    if (valid && rank == 0) cnt[w][d] = __popc(peers);
    __syncthreads();
    // exclusive prefix over warps for each digit (stable: lower warps first)
    if (t < 256) {
        int run = 0;
        for (int ww = 0; ww < kWarps; ++ww) {
            int v = cnt[ww][t];
            cnt[ww][t] = run;
            run += v;
        }
    }
    __syncthreads();
    if (valid) {
        int dst = offs[d * nblocks + blockIdx.x] + cnt[w][d] + rank;
        kout[dst] = key;
        vout[dst] = vin ? vin[i] : (int32_t)i;
    }
}

template <class W>
__global__ void count_adjacent_dups(const W *__restrict__ sorted, i64 n, int *__restrict__ flag) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (i < n && sorted[i] == sorted[i - 1]) atomicAdd(flag, 1);
}

template <class W>
int radix_sort(sbd_ctx *ctx, const W *keys, i64 n, int key_bits, DevBuf &sorted, DevBuf &perm) {
    cudaStream_t st = ctx->stream;
    SBD_CUDA(ctx, sorted.ensure(sizeof(W) * (n ? n : 1)));
    SBD_CUDA(ctx, perm.ensure(sizeof(int32_t) * (n ? n : 1)));
    if (n == 0) return SBD_OK;
    const int nblocks = (int)((n + kTile - 1) / kTile);
    DevBuf k2, v2, hist;
    SBD_CUDA(ctx, k2.ensure(sizeof(W) * n));
    SBD_CUDA(ctx, v2.ensure(sizeof(int32_t) * n));
    SBD_CUDA(ctx, hist.ensure(sizeof(int) * 256 * nblocks + 64));
    const int passes = std::max(1, (key_bits + 7) / 8);
    // ping-pong from caller order with identity values; the LAST pass lands in sorted/perm
    const W *kin = keys;
    const int32_t *vin = nullptr;
    W *bufk[2] = {sorted.as<W>(), k2.as<W>()};
    int32_t *bufv[2] = {perm.as<int32_t>(), v2.as<int32_t>()};
    int cur = (passes % 2 == 1) ? 0 : 1;
    for (int p = 0; p < passes; ++p) {
        radix_hist<W><<<nblocks, kTile, 0, st>>>(kin, n, 8 * p, hist.as<int>(), nblocks);
        exclusive_scan_small<<<1, 1024, 0, st>>>(hist.as<int>(), 256 * nblocks);
        radix_scatter<W><<<nblocks, kTile, 0, st>>>(kin, vin, bufk[cur], bufv[cur], n, 8 * p, hist.as<int>(), nblocks);
        SBD_LAUNCHED(ctx, "radix sort");
        kin = bufk[cur];
        vin = bufv[cur];
        cur ^= 1;
    }
    return SBD_OK;
}

template <class W>
int sort_strings(sbd_ctx *ctx, Sector &s, int norb) {
    const i64 n = s.n;
    cudaStream_t st = ctx->stream;
    int rc = radix_sort<W>(ctx, s.str.as<W>(), n, norb, s.sorted, s.perm);
    if (rc || n == 0) return rc;
    DevBuf flag;
    SBD_CUDA(ctx, flag.ensure(sizeof(int)));
    SBD_CUDA(ctx, cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    count_adjacent_dups<W><<<grid_for(n, 256), 256, 0, st>>>(s.sorted.as<W>(), n, flag.as<int>());
    SBD_LAUNCHED(ctx, "dup check");
    int dups = 0;
    SBD_CUDA(ctx, cudaMemcpyAsync(&dups, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    if (dups) return sbd_fail(ctx, SBD_EINVAL, "strings must be deduplicated");
    return SBD_OK;
}

}  // namespace

int sbd_radix_sort(sbd_ctx *ctx, const u64 *keys, i64 n, int key_bits, DevBuf &sorted, DevBuf &perm) {
    return radix_sort<u64>(ctx, keys, n, key_bits, sorted, perm);
}

int sbd_sort_strings(sbd_ctx *ctx, Sector &s) { return sort_strings<u64>(ctx, s, ctx->norb); }

int sbd_sort_strings128(sbd_ctx *ctx, Sector &s, int norb) { return sort_strings<U128>(ctx, s, norb); }
