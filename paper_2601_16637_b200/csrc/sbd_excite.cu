// Excitation generation on the device + kernel-ready coefficients.
//
// Reference semantics (bit-exact target):
//   enumerate_singles  basis.py:72-81   p occupied ascending, r virtual ascending
//   enumerate_doubles  basis.py:84-103  combinations(occ,2) x combinations(virt,2),
//                                       phase = sign(p->r on s) * sign(q->s on mid)
//   build_excitation_table basis.py:362-403: keep in-set targets only, CSR per
//                                       source string in caller order.
//
// Design: one warp per source string.  Lanes take consecutive candidates in
// enumeration order (32 per step), build the target mask, and look it up by
// binary search over the sorted sector (a shared-memory splitter level, then a
// short search in the L1-resident sorted array).  A ballot + popc compaction
// keeps enumeration order, so the count pass and the fill pass produce exactly
// the reference's entry order; targets are mapped back to caller indices
// through the sort permutation.  The kernel is templated on the string word
// (u64, or U128 for norb <= 128 -- sbd_table128_build, tables only).
#include <algorithm>
#include <cstdio>
#include <vector>

#include "sbd_internal.cuh"
#include "sbd_words.cuh"

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kSplit = 4096;  // splitter keys kept in shared memory

template <class W>
struct EnumSmem {
    static constexpr int kMaxOrb = 8 * (int)sizeof(W);
    static constexpr int kMaxPairs = kMaxOrb * (kMaxOrb - 1) / 2;
    W spl[kSplit];
    uint16_t hole_pairs[kMaxPairs];  // (a | a2 << 8) for a < a2 < n_occ, lexicographic
    uint16_t virt_pairs[kMaxPairs];
    uint8_t occ[kWarpsPerBlock][kMaxOrb];
    uint8_t virt[kWarpsPerBlock][kMaxOrb];
};

using words::sign_between;

// sorted position of key or -1
template <class W>
__device__ __forceinline__ int lookup(const EnumSmem<W> &sm, int nspl, int stride, const W *__restrict__ sorted,
                                      i64 n, W key) {
    // largest j with spl[j] <= key
    int lo = 0, hi = nspl;  // invariant answer in [lo-1, hi-1]
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (sm.spl[mid] <= key) lo = mid + 1;
        else hi = mid;
    }
    int j = lo - 1;
    if (j < 0) return -1;
    if (stride == 1) return sm.spl[j] == key ? j : -1;
    i64 a = (i64)j * stride, b = min(n, a + stride);
    while (a < b) {
        i64 mid = (a + b) >> 1;
        if (words::ldg(sorted + mid) < key) a = mid + 1;
        else b = mid;
    }
    return (a < n && words::ldg(sorted + a) == key) ? (int)a : -1;
}

template <bool FILL, class W>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
enum_kernel(const W *__restrict__ str, const W *__restrict__ sorted, const int32_t *__restrict__ perm, i64 n,
            int norb, int n_elec, int stride, int nspl,
            int64_t *__restrict__ cnt_s, int64_t *__restrict__ cnt_d,            // count pass: [n]
            const int64_t *__restrict__ s_off, const int64_t *__restrict__ d_off,  // fill pass
            int32_t *__restrict__ s_tgt, int16_t *__restrict__ s_hole, int16_t *__restrict__ s_part,
            int8_t *__restrict__ s_phase, int32_t *__restrict__ d_tgt, int16_t *__restrict__ d_h1,
            int16_t *__restrict__ d_h2, int16_t *__restrict__ d_p1, int16_t *__restrict__ d_p2,
            int8_t *__restrict__ d_phase) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    EnumSmem<W> &sm = *reinterpret_cast<EnumSmem<W> *>(smem_raw);
    const int no = n_elec, nv = norb - n_elec;
    const int nhp = no * (no - 1) / 2, nvp = nv * (nv - 1) / 2;
    for (int j = threadIdx.x; j < nspl; j += blockDim.x) sm.spl[j] = sorted[(i64)j * stride];
    for (int k = threadIdx.x; k < nhp; k += blockDim.x) {
        int a = 0, rem = k;
        while (rem >= no - a - 1) rem -= no - a - 1, ++a;
        sm.hole_pairs[k] = (uint16_t)(a | ((a + 1 + rem) << 8));
    }
    for (int k = threadIdx.x; k < nvp; k += blockDim.x) {
        int a = 0, rem = k;
        while (rem >= nv - a - 1) rem -= nv - a - 1, ++a;
        sm.virt_pairs[k] = (uint16_t)(a | ((a + 1 + rem) << 8));
    }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1;
    uint8_t *occ = sm.occ[w], *virt = sm.virt[w];
    for (i64 i = (i64)blockIdx.x * kWarpsPerBlock + w; i < n; i += (i64)gridDim.x * kWarpsPerBlock) {
        const W s = str[i];
        // occupied / virtual orbital lists in ascending order
        for (int base = 0; base < norb; base += 32) {
            int o = base + lane;
            bool in = o < norb, occd = in && words::test(s, o);
            unsigned mo = __ballot_sync(0xffffffffu, occd), mv = __ballot_sync(0xffffffffu, in && !occd);
            int before_o = words::popc_below(s, base);
            int before_v = base - before_o;
            if (occd) occ[before_o + __popc(mo & lt)] = (uint8_t)o;
            if (in && !occd) virt[before_v + __popc(mv & lt)] = (uint8_t)o;
        }
        __syncwarp();
        i64 ws = FILL ? s_off[i] : 0, wd = FILL ? d_off[i] : 0;
        // singles: candidate c -> (occ[c / nv], virt[c % nv])
        const int ts = no * nv;
        for (int base = 0; base < ts; base += 32) {
            int c = base + lane;
            int pos = -1, p = 0, r = 0;
            if (c < ts) {
                p = occ[c / nv];
                r = virt[c % nv];
                pos = lookup(sm, nspl, stride, sorted, n, words::move(s, p, r));
            }
            unsigned m = __ballot_sync(0xffffffffu, pos >= 0);
            if (FILL && pos >= 0) {
                i64 k = ws + __popc(m & lt);
                s_tgt[k] = perm[pos];
                s_hole[k] = (int16_t)p;
                s_part[k] = (int16_t)r;
                s_phase[k] = (int8_t)sign_between(s, p, r);
            }
            ws += __popc(m);
        }
        // doubles: candidate c -> hole pair c / nvp, particle pair c % nvp
        const i64 td = (i64)nhp * nvp;
        for (i64 base = 0; base < td; base += 32) {
            i64 c = base + lane;
            int pos = -1, p = 0, q = 0, r = 0, t = 0;
            W mid{};
            if (c < td) {
                uint16_t hp = sm.hole_pairs[c / nvp], vp = sm.virt_pairs[c % nvp];
                p = occ[hp & 0xFF];
                q = occ[hp >> 8];
                r = virt[vp & 0xFF];
                t = virt[vp >> 8];
                mid = words::move(s, p, r);
                pos = lookup(sm, nspl, stride, sorted, n, words::move(mid, q, t));
            }
            unsigned m = __ballot_sync(0xffffffffu, pos >= 0);
            if (FILL && pos >= 0) {
                i64 k = wd + __popc(m & lt);
                d_tgt[k] = perm[pos];
                d_h1[k] = (int16_t)p;
                d_h2[k] = (int16_t)q;
                d_p1[k] = (int16_t)r;
                d_p2[k] = (int16_t)t;
                d_phase[k] = (int8_t)(sign_between(s, p, r) * sign_between(mid, q, t));
            }
            wd += __popc(m);
        }
        if (!FILL && lane == 0) {
            cnt_s[i] = ws;
            cnt_d[i] = wd;
        }
        __syncwarp();
    }
}

// out[0] = 0, out[i+1] = sum_{j<=i} in[j]   (single block, n small)
__global__ void offsets_from_counts(const int64_t *__restrict__ in, int64_t *__restrict__ out, i64 n) {
    __shared__ int64_t part[1024];
    int t = threadIdx.x, nt = blockDim.x;
    i64 per = (n + nt - 1) / nt, lo = t * per, hi = min(n, lo + per);
    int64_t s = 0;
    for (i64 i = lo; i < hi; ++i) s += in[i];
    part[t] = s;
    __syncthreads();
    if (t == 0) {
        int64_t run = 0;
        for (int i = 0; i < nt; ++i) {
            int64_t v = part[i];
            part[i] = run;
            run += v;
        }
    }
    __syncthreads();
    int64_t run = part[t];
    if (t == 0) out[0] = 0;
    for (i64 i = lo; i < hi; ++i) {
        run += in[i];
        out[i + 1] = run;
    }
}

__device__ __forceinline__ double eri4(const double *__restrict__ eri, int p, int q, int r, int s) {
    return __ldg(eri + tri_idx(tri_idx(p, q), tri_idx(r, s)));
}

// Per source string: pack singles (with F = h_pr + sum_common[(pr|qq)-(pq|qr)],
// the spectator-free part of apply.py:115-134) and doubles (the full
// spectator-free element of apply.py:137-149) into Conn records; singles also
// into SConn records for the opposite-spin term; same-spin diagonal energy
// (apply.py:84-97) in the reference's operation order.
__global__ void coeff_kernel(const u64 *__restrict__ str, i64 n, int norb, const double *__restrict__ h,
                             const double *__restrict__ eri, const int64_t *__restrict__ s_off,
                             const int32_t *__restrict__ s_tgt, const int16_t *__restrict__ s_hole,
                             const int16_t *__restrict__ s_part, const int8_t *__restrict__ s_phase,
                             const int64_t *__restrict__ d_off, const int32_t *__restrict__ d_tgt,
                             const int16_t *__restrict__ d_h1, const int16_t *__restrict__ d_h2,
                             const int16_t *__restrict__ d_p1, const int16_t *__restrict__ d_p2,
                             const int8_t *__restrict__ d_phase, int64_t *__restrict__ conn_off,
                             Conn *__restrict__ conn, SConn *__restrict__ sconn, int32_t *__restrict__ s_row,
                             double *__restrict__ energy) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const u64 s = str[i];
    i64 base = s_off[i] + d_off[i];
    conn_off[i] = base;
    if (i == n - 1) conn_off[n] = s_off[n] + d_off[n];
    i64 o = base;
    for (i64 k = s_off[i]; k < s_off[i + 1]; ++k, ++o) {
        int p = s_hole[k], r = s_part[k], ph = s_phase[k];
        double F = __ldg(h + p * norb + r);
        for (u64 t = s & ~(1ull << p); t; t &= t - 1) {
            int q = __ffsll((long long)t) - 1;
            F = __dadd_rn(F, __dsub_rn(eri4(eri, p, r, q, q), eri4(eri, p, q, q, r)));
        }
        int P = (int)tri_idx(p, r);
        Conn c;
        c.tgt = s_tgt[k];
        c.info = ph * (P + 1);
        c.c = ph * F;
        conn[o] = c;
        SConn sc;
        sc.tgt = s_tgt[k];
        sc.info = ph * (P + 1);
        sconn[k] = sc;
        s_row[k] = (int32_t)i;
    }
    for (i64 k = d_off[i]; k < d_off[i + 1]; ++k, ++o) {
        int p = d_h1[k], q = d_h2[k], r = d_p1[k], t = d_p2[k];
        Conn c;
        c.tgt = d_tgt[k];
        c.info = 0;
        c.c = d_phase[k] * __dsub_rn(eri4(eri, p, r, q, t), eri4(eri, p, t, q, r));
        conn[o] = c;
    }
    double e = 0.0;
    for (u64 t = s; t; t &= t - 1) {
        int p = __ffsll((long long)t) - 1;
        e = __dadd_rn(e, __ldg(h + p * norb + p));
        for (u64 t2 = s; t2; t2 &= t2 - 1) {
            int q = __ffsll((long long)t2) - 1;
            e = __dadd_rn(e, __dmul_rn(0.5, __dsub_rn(eri4(eri, p, p, q, q), eri4(eri, p, q, q, p))));
        }
    }
    energy[i] = e;
}

// J[P][i] = sum_{q in string i, ascending} (P|qq)  -- spectator part of a single
__global__ void jtable_kernel(const u64 *__restrict__ str, i64 n, i64 npair, const double *__restrict__ eri,
                              double *__restrict__ J) {
    i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    i64 P = blockIdx.y;
    if (i >= n || P >= npair) return;
    double acc = 0.0;
    for (u64 t = str[i]; t; t &= t - 1) {
        int q = __ffsll((long long)t) - 1;
        acc = __dadd_rn(acc, __ldg(eri + tri_idx(P, tri_idx(q, q))));
    }
    J[P * n + i] = acc;
}

}  // namespace

// Sliced-ELL layout of the singles for the opposite-spin (task 0) kernel, built on the device.
//
// Strings are sorted by single count (descending, stable) into groups of 32
// positions.  The target index space [0, n) is cut into H chunks of
// sell_chunk strings; for chunk h, group g holds W_{h,g} slots (the widest
// position of the group), slot-major: entry q of position l at
// ent[goff[h][g] + 32 q + l].  An entry is packed as
//   (tgt - h * chunk) << sell_pbits | (P + neg * ld_vpp)
// i.e. the chunk-local target and the column of the sign-folded ERI row
// (sbd_context.cu: row (Pa, s_a) = [s_a (Pa|.), -s_a (Pa|.)]).  Unused slots
// point at local target `chunk`, a zero slot the kernel keeps after the
// staged chunk, so padding adds exactly 0.0 with no branch.  The layout only
// balances work and bank conflicts; it never changes which terms are summed.
namespace {

constexpr int kSellKeyChunks = 7;  // chunk counts in the sort key (after the 11-bit total)

// per string: singles per target chunk, and the sort key (total desc, then chunk counts desc)
__global__ void sell_count_kernel(i64 n, const int64_t *__restrict__ off, const SConn *__restrict__ sc, i64 H,
                                  i64 chunk, int32_t *__restrict__ cc, u64 *__restrict__ key) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (i64 h = 0; h < H; ++h) cc[i * H + h] = 0;
    for (i64 k = off[i]; k < off[i + 1]; ++k) ++cc[i * H + sc[k].tgt / chunk];
    const i64 tot = min(off[i + 1] - off[i], (i64)2047);
    u64 kk = (u64)(2047 - tot);
    const i64 hk = H < kSellKeyChunks ? H : kSellKeyChunks;
    for (i64 h = 0; h < hk; ++h) kk = (kk << 7) | (u64)(127 - min(cc[i * H + h], 127));
    key[i] = kk;
}

// W_{h,g} = widest position of group g in chunk h, as a slot count x 32
__global__ void sell_width_kernel(i64 n, i64 H, i64 groups, const int32_t *__restrict__ cc,
                                  const int32_t *__restrict__ order, int64_t *__restrict__ wcount) {
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= H * groups) return;
    const i64 h = t / groups, g = t % groups;
    int32_t w = 0;
    for (i64 l = 0; l < 32 && g * 32 + l < n; ++l) w = max(w, cc[(i64)order[g * 32 + l] * H + h]);
    wcount[t] = 32 * (int64_t)w;
}

// goff[h][g] (int32, groups + 1 per chunk) from the flat exclusive scan over (h, g)
__global__ void sell_goff_kernel(i64 H, i64 groups, const int64_t *__restrict__ flat, int32_t *__restrict__ goff) {
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= H * (groups + 1)) return;
    const i64 h = t / (groups + 1), g = t % (groups + 1);
    goff[t] = (int32_t)flat[h * groups + g];
}

__global__ void sell_col_kernel(i64 n, i64 groups, const int32_t *__restrict__ order, int32_t *__restrict__ col) {
    const i64 p = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < groups * 32) col[p] = p < n ? order[p] : -1;
}

// Distinct shared-memory addresses per 64-bit bank of one half-warp slot (<= 16 addresses in all).
struct BankSet {
    int64_t addr[16];
    int n = 0;
    __device__ int load(int64_t a) const {  // wavefronts of a's bank if a were added
        int same = 0;
        bool present = false;
        for (int i = 0; i < n; ++i)
            if ((addr[i] & 15) == (a & 15)) {
                ++same;
                present |= addr[i] == a;
            }
        return same + (present ? 0 : 1);
    }
    __device__ void add(int64_t a) {
        for (int i = 0; i < n; ++i)
            if (addr[i] == a) return;
        addr[n++] = a;
    }
    __device__ int maxload() const {
        int m = 0;
        for (int i = 0; i < n; ++i) {
            int c = 0;
            for (int j = 0; j < n; ++j) c += (addr[j] & 15) == (addr[i] & 15) && (j == i || addr[j] != addr[i]);
            m = max(m, c);
        }
        return m;
    }
};

constexpr int kSellGreedyMax = 32;  // widest slot count the greedy assignment handles (wider: enumeration order)

// One thread per (group, chunk).  A position's singles may sit in its slots in any order (the sum
// is the same up to rounding), so each slot's 32 entries can be chosen to spread the two
// shared-memory gathers of the task-0 inner loop -- x[jl] and the ERI row at (chunk + 2 + q) --
// over the 16 64-bit banks of each half-warp.  Cost model: per half-warp and slot, a gather takes
// as many wavefronts as the most-loaded bank has DISTINCT addresses (equal addresses broadcast).
// The table keeps the better of the enumeration order and a greedy assignment (per lane, the
// remaining entry that adds the fewest wavefronts).
__global__ void sell_fill_kernel(i64 n, i64 H, i64 groups, i64 chunk, int pbits, i64 ldv,
                                 const int64_t *__restrict__ off, const SConn *__restrict__ sc,
                                 const int32_t *__restrict__ order, const int32_t *__restrict__ goff,
                                 uint32_t *__restrict__ ent) {
    const i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= H * groups) return;
    const i64 g = t / H, h = t % H;
    const i64 base = goff[h * (groups + 1) + g];
    const i64 w = (goff[h * (groups + 1) + g + 1] - base) / 32;
    if (w == 0) return;
    const uint32_t null_ent = (uint32_t)chunk << pbits, qmask = (1u << pbits) - 1u;
    auto entry = [&](int l, i64 q) -> uint32_t {  // q-th single of position l inside chunk h (enumeration order)
        const i64 p = g * 32 + l;
        if (p >= n) return null_ent;
        const int32_t c = order[p];
        i64 seen = 0;
        for (i64 k = off[c]; k < off[c + 1]; ++k) {
            if (sc[k].tgt / chunk != h) continue;
            if (seen++ == q) {
                const i64 jl = sc[k].tgt - h * chunk;
                const i64 P = abs(sc[k].info) - 1, neg = sc[k].info < 0;
                return ((uint32_t)jl << pbits) | (uint32_t)(P + neg * ldv);
            }
        }
        return null_ent;
    };
    auto xaddr = [&](uint32_t e) { return (int64_t)(e >> pbits); };
    auto vaddr = [&](uint32_t e) { return (int64_t)(chunk + 2 + (e & qmask)); };
    // enumeration order and its cost
    int cost_nat = 0;
    for (i64 q = 0; q < w; ++q)
        for (int half = 0; half < 2; ++half) {
            BankSet bx, bv;
            for (int l = 16 * half; l < 16 * half + 16; ++l) {
                const uint32_t e = entry(l, q);
                if (e == null_ent) continue;
                bx.add(xaddr(e));
                bv.add(vaddr(e));
            }
            cost_nat += bx.maxload() + bv.maxload();
        }
    bool greedy = false;
    if (w <= kSellGreedyMax) {
        // greedy assignment, written straight into the table; kept if cheaper
        uint32_t rem[16][kSellGreedyMax];
        int nrem[16];
        int cost_gr = 0;
        for (int half = 0; half < 2; ++half) {
            for (int l = 0; l < 16; ++l) {
                nrem[l] = 0;
                for (i64 q = 0; q < w; ++q) {
                    const uint32_t e = entry(16 * half + l, q);
                    if (e != null_ent) rem[l][nrem[l]++] = e;
                }
            }
            for (i64 q = 0; q < w; ++q) {
                BankSet bx, bv;
                for (int l = 0; l < 16; ++l) {
                    uint32_t e = null_ent;
                    if (nrem[l] > 0) {
                        int best = 0, best_cost = 1 << 30;
                        for (int k = 0; k < nrem[l]; ++k) {
                            const int lx = bx.load(xaddr(rem[l][k])), lv = bv.load(vaddr(rem[l][k]));
                            const int cost = 4 * max(lx, lv) + lx + lv;
                            if (cost < best_cost) {
                                best_cost = cost;
                                best = k;
                            }
                        }
                        e = rem[l][best];
                        rem[l][best] = rem[l][--nrem[l]];
                        bx.add(xaddr(e));
                        bv.add(vaddr(e));
                    }
                    ent[base + 32 * q + 16 * half + l] = e;
                }
                cost_gr += bx.maxload() + bv.maxload();
            }
        }
        greedy = cost_gr < cost_nat;
    }
    if (!greedy)
        for (i64 q = 0; q < w; ++q)
            for (int l = 0; l < 32; ++l) ent[base + 32 * q + l] = entry(l, q);
}

}  // namespace

static int build_sell(sbd_ctx *ctx, Sector &s) {
    const i64 n = s.n;
    cudaStream_t st = ctx->stream;
    const i64 H = n <= kSellWhole ? 1 : (n + kSellChunk - 1) / kSellChunk;
    const i64 chunk = std::max<i64>(2, ((n + H - 1) / H + 1) & ~(i64)1);  // even: 16-byte TMA rows
    int pbits = 1;
    while (((i64)1 << pbits) < 2 * ctx->ld_vpp) ++pbits;
    int cbits = 1;
    while (((i64)1 << cbits) <= chunk) ++cbits;
    if (pbits + cbits > 32) return sbd_fail(ctx, SBD_EINVAL, "sector too large for the packed single-excitation table");
    const i64 groups = (n + 31) / 32;
    DevBuf cc, key, skey, order, wcount, flat;
    SBD_CUDA(ctx, cc.ensure(sizeof(int32_t) * std::max<i64>(1, n * H)));
    SBD_CUDA(ctx, key.ensure(sizeof(u64) * std::max<i64>(1, n)));
    sell_count_kernel<<<grid_for(n, 128), 128, 0, st>>>(n, s.s_off.as<int64_t>(), s.sconn.as<SConn>(), H, chunk,
                                                        cc.as<int32_t>(), key.as<u64>());
    SBD_LAUNCHED(ctx, "sell counts");
    // stable sort by (total, per-chunk counts) descending: padding stays small in every chunk
    int rc = sbd_radix_sort(ctx, key.as<u64>(), n, 11 + 7 * (int)std::min<i64>(H, kSellKeyChunks), skey, order);
    if (rc) return rc;
    SBD_CUDA(ctx, wcount.ensure(sizeof(int64_t) * std::max<i64>(1, H * groups)));
    SBD_CUDA(ctx, flat.ensure(sizeof(int64_t) * (H * groups + 1)));
    sell_width_kernel<<<grid_for(H * groups, 128), 128, 0, st>>>(n, H, groups, cc.as<int32_t>(), order.as<int32_t>(),
                                                                 wcount.as<int64_t>());
    offsets_from_counts<<<1, 1024, 0, st>>>(wcount.as<int64_t>(), flat.as<int64_t>(), H * groups);
    SBD_LAUNCHED(ctx, "sell widths");
    int64_t total = 0;
    SBD_CUDA(ctx, cudaMemcpyAsync(&total, flat.as<int64_t>() + H * groups, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    if (total >= (int64_t)INT32_MAX) return sbd_fail(ctx, SBD_EINVAL, "singles table too large");
    SBD_CUDA(ctx, s.sell_ent.ensure(sizeof(uint32_t) * (total + 4)));
    SBD_CUDA(ctx, s.sell_goff.ensure(sizeof(int32_t) * H * (groups + 1)));
    SBD_CUDA(ctx, s.sell_col.ensure(sizeof(int32_t) * (groups * 32 + 1)));
    sell_goff_kernel<<<grid_for(H * (groups + 1), 128), 128, 0, st>>>(H, groups, flat.as<int64_t>(),
                                                                     s.sell_goff.as<int32_t>());
    sell_col_kernel<<<grid_for(groups * 32, 128), 128, 0, st>>>(n, groups, order.as<int32_t>(), s.sell_col.as<int32_t>());
    sell_fill_kernel<<<grid_for(H * groups, 64), 64, 0, st>>>(n, H, groups, chunk, pbits, ctx->ld_vpp,
                                                               s.s_off.as<int64_t>(), s.sconn.as<SConn>(),
                                                               order.as<int32_t>(), s.sell_goff.as<int32_t>(),
                                                               s.sell_ent.as<uint32_t>());
    SBD_LAUNCHED(ctx, "sell fill");
    const uint32_t pad[4] = {(uint32_t)chunk << pbits, (uint32_t)chunk << pbits, (uint32_t)chunk << pbits,
                             (uint32_t)chunk << pbits};
    SBD_CUDA(ctx, cudaMemcpyAsync(s.sell_ent.as<uint32_t>() + total, pad, sizeof(pad), cudaMemcpyHostToDevice, st));
    s.sell_goff_host.resize((size_t)(H * (groups + 1)));
    SBD_CUDA(ctx, cudaMemcpyAsync(s.sell_goff_host.data(), s.sell_goff.p, sizeof(int32_t) * s.sell_goff_host.size(),
                                  cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    s.sell_groups = groups;
    s.sell_nent = total;
    s.sell_h = H;
    s.sell_chunk = chunk;
    s.sell_pbits = pbits;
    return SBD_OK;
}

namespace {

template <class W>
int build_tables(sbd_ctx *ctx, Sector &s, int norb) {
    const i64 n = s.n;
    cudaStream_t st = ctx->stream;
    SBD_CUDA(ctx, s.s_off.ensure(sizeof(int64_t) * (n + 1)));
    SBD_CUDA(ctx, s.d_off.ensure(sizeof(int64_t) * (n + 1)));
    if (n == 0) {
        SBD_CUDA(ctx, cudaMemsetAsync(s.s_off.p, 0, sizeof(int64_t), st));
        SBD_CUDA(ctx, cudaMemsetAsync(s.d_off.p, 0, sizeof(int64_t), st));
        s.ns = s.nd = 0;
        return SBD_OK;
    }
    int stride = (int)((n + kSplit - 1) / kSplit);
    int nspl = (int)((n + stride - 1) / stride);
    DevBuf cs, cd;
    SBD_CUDA(ctx, cs.ensure(sizeof(int64_t) * n));
    SBD_CUDA(ctx, cd.ensure(sizeof(int64_t) * n));
    size_t smem = sizeof(EnumSmem<W>);
    SBD_CUDA(ctx, cudaFuncSetAttribute(enum_kernel<false, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SBD_CUDA(ctx, cudaFuncSetAttribute(enum_kernel<true, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    unsigned blocks = (unsigned)std::min<i64>((n + kWarpsPerBlock - 1) / kWarpsPerBlock, (i64)ctx->num_sms * 8);
    enum_kernel<false, W><<<blocks, kWarpsPerBlock * 32, smem, st>>>(
        s.str.as<W>(), s.sorted.as<W>(), s.perm.as<int32_t>(), n, norb, s.n_elec, stride, nspl,
        cs.as<int64_t>(), cd.as<int64_t>(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
        nullptr, nullptr, nullptr, nullptr);
    SBD_LAUNCHED(ctx, "enum count");
    offsets_from_counts<<<1, 1024, 0, st>>>(cs.as<int64_t>(), s.s_off.as<int64_t>(), n);
    offsets_from_counts<<<1, 1024, 0, st>>>(cd.as<int64_t>(), s.d_off.as<int64_t>(), n);
    SBD_LAUNCHED(ctx, "enum offsets");
    int64_t tot[2];
    SBD_CUDA(ctx, cudaMemcpyAsync(&tot[0], s.s_off.as<int64_t>() + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaMemcpyAsync(&tot[1], s.d_off.as<int64_t>() + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    s.ns = tot[0];
    s.nd = tot[1];
    if (s.ns + s.nd >= (i64)INT32_MAX) return sbd_fail(ctx, SBD_EINVAL, "excitation table too large");
    SBD_CUDA(ctx, s.s_tgt.ensure(sizeof(int32_t) * (s.ns + 1)));
    SBD_CUDA(ctx, s.s_hole.ensure(sizeof(int16_t) * (s.ns + 1)));
    SBD_CUDA(ctx, s.s_part.ensure(sizeof(int16_t) * (s.ns + 1)));
    SBD_CUDA(ctx, s.s_phase.ensure(sizeof(int8_t) * (s.ns + 1)));
    SBD_CUDA(ctx, s.d_tgt.ensure(sizeof(int32_t) * (s.nd + 1)));
    SBD_CUDA(ctx, s.d_h1.ensure(sizeof(int16_t) * (s.nd + 1)));
    SBD_CUDA(ctx, s.d_h2.ensure(sizeof(int16_t) * (s.nd + 1)));
    SBD_CUDA(ctx, s.d_p1.ensure(sizeof(int16_t) * (s.nd + 1)));
    SBD_CUDA(ctx, s.d_p2.ensure(sizeof(int16_t) * (s.nd + 1)));
    SBD_CUDA(ctx, s.d_phase.ensure(sizeof(int8_t) * (s.nd + 1)));
    enum_kernel<true, W><<<blocks, kWarpsPerBlock * 32, smem, st>>>(
        s.str.as<W>(), s.sorted.as<W>(), s.perm.as<int32_t>(), n, norb, s.n_elec, stride, nspl, nullptr,
        nullptr, s.s_off.as<int64_t>(), s.d_off.as<int64_t>(), s.s_tgt.as<int32_t>(), s.s_hole.as<int16_t>(),
        s.s_part.as<int16_t>(), s.s_phase.as<int8_t>(), s.d_tgt.as<int32_t>(), s.d_h1.as<int16_t>(),
        s.d_h2.as<int16_t>(), s.d_p1.as<int16_t>(), s.d_p2.as<int16_t>(), s.d_phase.as<int8_t>());
    SBD_LAUNCHED(ctx, "enum fill");
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    return SBD_OK;
}

}  // namespace

int sbd_build_sector_tables(sbd_ctx *ctx, Sector &s) { return build_tables<u64>(ctx, s, ctx->norb); }

int sbd_build_sector_tables128(sbd_ctx *ctx, Sector &s, int norb) { return build_tables<U128>(ctx, s, norb); }

int sbd_build_coefficients(sbd_ctx *ctx, Sector &s, const Sector &other) {
    (void)other;
    const i64 n = s.n;
    cudaStream_t st = ctx->stream;
    SBD_CUDA(ctx, s.conn_off.ensure(sizeof(int64_t) * (n + 1)));
    SBD_CUDA(ctx, s.conn.ensure(sizeof(Conn) * (s.ns + s.nd + 1)));
    SBD_CUDA(ctx, s.sconn.ensure(sizeof(SConn) * (s.ns + 1)));
    SBD_CUDA(ctx, s.s_row.ensure(sizeof(int32_t) * (s.ns + 1)));
    SBD_CUDA(ctx, s.energy.ensure(sizeof(double) * (n + 1)));
    SBD_CUDA(ctx, s.J.ensure(sizeof(double) * (ctx->npair * n + 1)));
    if (n == 0) {
        SBD_CUDA(ctx, cudaMemsetAsync(s.conn_off.p, 0, sizeof(int64_t), st));
        return SBD_OK;
    }
    coeff_kernel<<<grid_for(n, 128), 128, 0, st>>>(
        s.str.as<u64>(), n, ctx->norb, ctx->h.as<double>(), ctx->eri.as<double>(), s.s_off.as<int64_t>(),
        s.s_tgt.as<int32_t>(), s.s_hole.as<int16_t>(), s.s_part.as<int16_t>(), s.s_phase.as<int8_t>(),
        s.d_off.as<int64_t>(), s.d_tgt.as<int32_t>(), s.d_h1.as<int16_t>(), s.d_h2.as<int16_t>(),
        s.d_p1.as<int16_t>(), s.d_p2.as<int16_t>(), s.d_phase.as<int8_t>(), s.conn_off.as<int64_t>(),
        s.conn.as<Conn>(), s.sconn.as<SConn>(), s.s_row.as<int32_t>(), s.energy.as<double>());
    SBD_LAUNCHED(ctx, "coefficients");
    dim3 g(grid_for(n, 128), (unsigned)ctx->npair);
    jtable_kernel<<<g, 128, 0, st>>>(s.str.as<u64>(), n, ctx->npair, ctx->eri.as<double>(), s.J.as<double>());
    SBD_LAUNCHED(ctx, "jtable");
#ifdef SBD_TIMING
    cudaStreamSynchronize(st);
    fprintf(stderr, "[sbd timing] (coefficients + J done; SELL next)\n");
#endif
    // packed singles for the opposite-spin (task 0) kernel
    if (n >= kPackMaxStrings || ctx->npair >= ((i64)1 << kPackPairBits))
        return sbd_fail(ctx, SBD_EINVAL, "sector too large for the packed single-excitation table");
    return build_sell(ctx, s);
    return SBD_OK;
}
