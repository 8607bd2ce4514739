// Task 0 in the dense regime as a contraction on the fp64 tensor cores.
//
// Reference: the alpha-single x beta-single opposite-spin doubles of
// _product_row (apply.py:228-238):
//   sigma[ia, ib] += sum_{k in aS(ia)} sum_{m in bS(ib)} s_k s_m (Pa_k | Pb_m) X[ja_k, jb_m]
//
// The SELL kernels (sbd_sigma.cu) evaluate that sum term by term: one shared
// load, two shared gathers and one FMA per (k, m) pair, 36 x 36 = 1296 terms
// per determinant for the full 12-orbital set.  When most candidate beta
// singles are in the set (the full string space, cfg1), the same sum factors
// through the pair index (the direct-CI form):
//   G[q][jb]     = sum_k  s_k (Pa_k | Q_q) X[ja_k, jb]          (a GEMM, K = |aS(ia)|)
//   sigma[ia,ib] = sum_m  s_m G[q(Pb_m)][jb_m]                  (36 gathers per determinant)
// with q over the norb (norb - 1) / 2 off-diagonal orbital pairs.
//
// Kernel: one persistent CTA per SM (16 warps) walks its alpha rows; a row's beta
// columns jb are cut into tiles of 128.  Per (row, tile):
//   1. the row's K x 128 slab of x (rows ja_k) is staged by cp.async, one
//      tile ahead (double buffer), with the tile's gather block (below);
//   2. G tile (nqp x 128) = E (nqp x Kp, built once per row from the pair-pair
//      ERI matrix and the alpha phases; each warp keeps its fragments of it in
//      registers for the whole row) times the slab, on DMMA.8x8x4: the warps
//      form a 4 x 4 grid over row fragments x 32-column quarters;
//   3. each thread owns beta positions ib and adds, in a fixed order, the G
//      entries its beta singles point at inside this tile (a u16 ELL block per
//      tile, staged in shared memory; padding reads a zero row of G): no
//      atomics, bitwise reproducible.
// The row is written once (or added, for the additive task-0 order).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "sbd_internal.cuh"
#include "sbd_ptx.cuh"

namespace {

constexpr int kDciThreads = 512;          // 16 warps, one CTA per SM
constexpr int kMaxSingles = 64;           // beta singles per string handled by the list builder
constexpr size_t kDciSmemMax = 227 * 1024;
// Tile of kNT = 128 beta columns.  The 16 warps form a 4 x 4 grid over (row fragments, column
// fragments): warp (mg, ng) owns row fragments m = mg + 4 j and the four column fragments
// 4 ng .. 4 ng + 3, and keeps its E fragments in registers for the whole alpha row (E changes per
// row, the slab per tile): a k-step costs 4 shared loads for 4 MFW DMMAs.
constexpr int kNT = 128;
constexpr int kLdX = kNT + 4;    // slab row stride (doubles): B-fragment loads conflict-free
constexpr int kLdG = kNT + 8;    // G row stride: C-fragment double2 stores conflict-free
constexpr int kNFW = 4;          // column fragments per warp
constexpr int kMG = 4;           // warp groups along the row fragments

struct DciArgs {
    i64 n_rows, row_base, nb;
    const double *X;
    double *Y;
    const int64_t *a_s_off;
    const SConn *a_sconn;
    const double *eq;        // [npair][nqp]: (P | Q_q), zero for q >= nq
    int nqp, kp_max, ld_e;   // ld_e = 4 (mod 16) doubles: A-fragment loads conflict-free
    // beta singles for the gather, per column tile t an ELL block [w_t][nb] at ell + woff[t]:
    // u16 entry (jb - t NT) << 8 | q << 1 | neg; padding points at the zero row q = nqp (< 128) of G
    const uint16_t *ell;
    const int64_t *woff;
    const int32_t *wt;
    int ntiles;
    int wmax;                // widest tile block (its [wmax][nb] u16 is staged into shared memory)
    bool add;
};

// E, the slab (double-buffered), G (nqp rows + the zero row) and one tile's ELL block
__host__ __device__ inline size_t dci_smem(int nqp, int kp_max, int ld_e, i64 ell_entries = 0) {
    return sizeof(double) * ((size_t)nqp * ld_e + 2 * (size_t)kp_max * kLdX + (size_t)(nqp + 1) * kLdG) +
           sizeof(uint16_t) * (size_t)((ell_entries + 7) & ~(i64)7);
}
__host__ __device__ inline int dci_ld_e(int kp) { return kp + (((4 - kp) % 16) + 16) % 16; }

// Stage rows ja_k (k < K) of x, columns [t NT, t NT + NT), into `xs`; rows K..Kp-1 and
// columns past nb are zero (E is zero there too, but the slab must not hold NaNs).
__device__ __forceinline__ void dci_stage(const DciArgs &a, double *xs, i64 row, int t, int K, int Kp) {
    const i64 e0 = a.a_s_off[row];
    const i64 c0 = (i64)t * kNT;
    const int cols = (int)min((i64)kNT, a.nb - c0);
    constexpr int kChunks = kNT / 2;  // 16-byte chunks per slab row
    for (int c = threadIdx.x; c < Kp * kChunks; c += kDciThreads) {
        const int k = c / kChunks, j = c % kChunks;
        double *dst = xs + k * kLdX + 2 * j;
        if (k < K && 2 * j < cols) {
            const i64 ja = a.a_sconn[e0 + k].tgt;
            cp_async16(dst, a.X + ja * a.nb + c0 + 2 * j);
        } else {
            *reinterpret_cast<double2 *>(dst) = make_double2(0.0, 0.0);
        }
    }
}

// tile t's ELL block [wt][nb] (contiguous in global memory) into shared memory, 16-byte copies
__device__ __forceinline__ void dci_stage_ell(const DciArgs &a, uint16_t *es_ell, int t) {
    // blocks are padded to 8 entries (16 bytes) in global memory, so whole 16-byte chunks copy
    const i64 chunks = ((i64)__ldg(a.wt + t) * a.nb + 7) / 8, base = __ldg(a.woff + t);
    const uint16_t *src = a.ell + base;
    for (i64 c = threadIdx.x; c < chunks; c += kDciThreads) cp_async16(es_ell + 8 * c, src + 8 * c);
}

// next row of this CTA that has alpha singles (n_rows if none)
__device__ __forceinline__ i64 dci_next_row(const DciArgs &a, i64 r) {
    for (; r < a.n_rows; r += gridDim.x)
        if (a.a_s_off[a.row_base + r + 1] > a.a_s_off[a.row_base + r]) return r;
    return a.n_rows;
}

// MFW: row fragments per warp (ceil(nqp / 8 / kMG)); KS: k-steps held in registers (Kp / 4 <= KS)
template <int MFW, int KS, int PPT>
__global__ void __launch_bounds__(kDciThreads, 1) cross_kernel_dci(DciArgs a) {
    extern __shared__ __align__(128) unsigned char dsm[];
    double *es = reinterpret_cast<double *>(dsm);     // [nqp][ld_e]
    double *xs0 = es + (size_t)a.nqp * a.ld_e;        // 2 x [kp_max][kLdX]
    double *gs = xs0 + 2 * (size_t)a.kp_max * kLdX;   // [nqp + 1][kLdG], row nqp = 0
    uint16_t *els = reinterpret_cast<uint16_t *>(gs + (size_t)(a.nqp + 1) * kLdG);  // [wt][nb] of the tile
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mg = warp / kMG, ng = warp % kMG;
    const int mf = a.nqp / 8;

    i64 r = dci_next_row(a, blockIdx.x);
    if (r >= a.n_rows) return;
    for (int c = threadIdx.x; c < kNT; c += kDciThreads) gs[a.nqp * kLdG + c] = 0.0;  // the padding row
    auto kof = [&](i64 rr) { return (int)(a.a_s_off[a.row_base + rr + 1] - a.a_s_off[a.row_base + rr]); };
    int K = kof(r), Kp = (K + 3) & ~3;
    int t = 0, buf = 0;
    dci_stage(a, xs0, a.row_base + r, 0, K, Kp);
    cp_async_commit();
    dci_stage_ell(a, els, 0);
    cp_async_commit();

    double acc[PPT];
#pragma unroll
    for (int i = 0; i < PPT; ++i) acc[i] = 0.0;
    double af[MFW][KS];  // this warp's E fragments for the current row

    while (true) {
        // the item after this one: next tile of the row, else tile 0 of the CTA's next row
        i64 rn = r;
        int tn = t + 1;
        if (tn == a.ntiles) {
            rn = dci_next_row(a, r + gridDim.x);
            tn = 0;
        }
        const int Kn = rn < a.n_rows ? kof(rn) : 0, Kpn = (Kn + 3) & ~3;
        if (rn < a.n_rows) dci_stage(a, xs0 + (size_t)(buf ^ 1) * a.kp_max * kLdX, a.row_base + rn, tn, Kn, Kpn);
        cp_async_commit();
        if (t == 0) {  // E for this row: E[q][k] = s_k (Pa_k | Q_q); the previous row's GEMM is done
            const i64 e0 = a.a_s_off[a.row_base + r];
            for (int i = threadIdx.x; i < a.nqp * Kp; i += kDciThreads) {
                const int q = i / Kp, k = i % Kp;
                double v = 0.0;
                if (k < K) {
                    const SConn sa = a.a_sconn[e0 + k];
                    v = __ldg(a.eq + (i64)(abs(sa.info) - 1) * a.nqp + q);
                    if (sa.info < 0) v = -v;
                }
                es[q * a.ld_e + k] = v;
            }
        }
        const int wt = __ldg(a.wt + t);
        cp_async_wait<1>();  // everything but the next item's slab: this slab and this tile's ELL block
        __syncthreads();  // slab `buf`, E and the ELL block visible; the previous gather is done with G
        if (t == 0) {     // E fragments of this warp into registers, for all tiles of the row
            const double *ap = es + (mg * 8 + (lane >> 2)) * a.ld_e + (lane & 3);
#pragma unroll
            for (int j = 0; j < MFW; ++j)
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
                    af[j][ks] = (mg + kMG * j < mf && 4 * ks < Kp) ? ap[j * kMG * 8 * a.ld_e + 4 * ks] : 0.0;
        }

        // G tile = E (nqp x Kp) * slab (Kp x NT)
        {
            const double *xs = xs0 + (size_t)buf * a.kp_max * kLdX;
            double d[MFW][kNFW][2];
#pragma unroll
            for (int j = 0; j < MFW; ++j)
#pragma unroll
                for (int n = 0; n < kNFW; ++n) d[j][n][0] = d[j][n][1] = 0.0;
            const double *bp = xs + (lane & 3) * kLdX + ng * (8 * kNFW) + (lane >> 2);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                if (4 * ks < Kp) {
                    double b[kNFW];
#pragma unroll
                    for (int n = 0; n < kNFW; ++n) b[n] = bp[4 * ks * kLdX + 8 * n];
#pragma unroll
                    for (int j = 0; j < MFW; ++j)
                        if (mg + kMG * j < mf)
#pragma unroll
                            for (int n = 0; n < kNFW; ++n) dmma_8x8x4(d[j][n][0], d[j][n][1], af[j][ks], b[n]);
                }
            }
#pragma unroll
            for (int j = 0; j < MFW; ++j) {
                const int m = mg + kMG * j;
                if (m < mf)
#pragma unroll
                    for (int n = 0; n < kNFW; ++n)
                        *reinterpret_cast<double2 *>(gs + (m * 8 + (lane >> 2)) * kLdG + ng * (8 * kNFW) + 8 * n +
                                                     2 * (lane & 3)) = make_double2(d[j][n][0], d[j][n][1]);
            }
        }
        __syncthreads();  // G tile complete

        // gather: sigma[ib] += s_m G[q_m][jb_m] for the beta singles of ib that land in tile t
        // (ELL slots of the tile from shared memory, padding reads the zero row)
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const i64 ib = threadIdx.x + (i64)i * kDciThreads;
            if (ib < a.nb) {
                const uint16_t *ep = els + ib;
                double s = acc[i];
                for (int sl = 0; sl < wt; ++sl) {
                    const uint32_t u = ep[(i64)sl * a.nb];
                    const double g = gs[((u >> 1) & 0x7fu) * kLdG + (u >> 8)];
                    s += (u & 1u) ? -g : g;
                }
                acc[i] = s;
            }
        }
        __syncthreads();  // every thread is done with this tile's ELL block
        if (rn < a.n_rows) dci_stage_ell(a, els, tn);  // the next item's block, in flight over its GEMM
        cp_async_commit();
        if (t == a.ntiles - 1) {
            double *yr = a.Y + r * a.nb;
#pragma unroll
            for (int i = 0; i < PPT; ++i) {
                const i64 ib = threadIdx.x + (i64)i * kDciThreads;
                if (ib < a.nb) {
                    if (a.add) yr[ib] += acc[i];
                    else yr[ib] = acc[i];
                }
                acc[i] = 0.0;
            }
        }
        if (rn >= a.n_rows) break;
        r = rn;
        t = tn;
        K = Kn;
        Kp = Kpn;
        buf ^= 1;
    }
    cp_async_wait<0>();
}

// Per beta string: its in-set singles sorted by target, packed for the gather, and the
// first entry of every column tile.
__global__ void dci_lists_kernel(i64 nb, const int64_t *__restrict__ s_off, const SConn *__restrict__ sconn,
                                 const int32_t *__restrict__ qmap, int nt, int ntiles, uint32_t *__restrict__ ent,
                                 int32_t *__restrict__ toff) {
    const i64 ib = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (ib >= nb) return;
    const i64 s0 = s_off[ib];
    const int n = (int)(s_off[ib + 1] - s0);
    int32_t tg[kMaxSingles];
    uint32_t code[kMaxSingles];
    for (int i = 0; i < n; ++i) {
        const SConn sc = sconn[s0 + i];
        const int32_t jb = sc.tgt;
        const uint32_t c = ((uint32_t)qmap[abs(sc.info) - 1] << 1) | (sc.info < 0 ? 1u : 0u);
        int j = i;
        while (j > 0 && tg[j - 1] > jb) {
            tg[j] = tg[j - 1];
            code[j] = code[j - 1];
            --j;
        }
        tg[j] = jb;
        code[j] = c;
    }
    int i = 0;
    for (int t = 0; t <= ntiles; ++t) {
        while (i < n && tg[i] < t * nt) ++i;
        toff[ib * (ntiles + 1) + t] = (int32_t)(s0 + i);
    }
    for (int k = 0; k < n; ++k) ent[s0 + k] = ((uint32_t)(tg[k] % nt) << 16) | code[k];
}

// ELL width of tile t: the most singles any beta string has into it
__global__ void dci_width_kernel(i64 nb, const int32_t *__restrict__ toff, int ntiles, int32_t *__restrict__ wt) {
    const i64 ib = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (ib >= nb) return;
    for (int t = 0; t < ntiles; ++t) atomicMax(wt + t, toff[ib * (ntiles + 1) + t + 1] - toff[ib * (ntiles + 1) + t]);
}

// tile-major u16 ELL blocks: slot s of string ib in tile t at ell[woff[t] + s nb + ib], padded with `pad`;
// ent holds (jb - t NT) << 16 | q << 1 | neg, re-packed as (jb - t NT) << 8 | q << 1 | neg
__global__ void dci_ell_kernel(i64 nb, const int32_t *__restrict__ toff, const uint32_t *__restrict__ ent, int ntiles,
                               const int32_t *__restrict__ wt, const int64_t *__restrict__ woff, uint32_t pad,
                               uint16_t *__restrict__ ell) {
    const i64 ib = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (ib >= nb) return;
    for (int t = 0; t < ntiles; ++t) {
        const int lo = toff[ib * (ntiles + 1) + t], cnt = toff[ib * (ntiles + 1) + t + 1] - lo;
        for (int sl = 0; sl < wt[t]; ++sl) {
            const uint32_t e = sl < cnt ? ent[lo + sl] : pad;
            ell[woff[t] + (i64)sl * nb + ib] = (uint16_t)(((e >> 16) << 8) | (e & 0xffu));
        }
    }
}

// eq[P][q] = (P | Q_q) over the off-diagonal pairs Q_q, zero for q >= nq
__global__ void dci_eq_kernel(i64 npair, int nq, int nqp, const int32_t *__restrict__ qpair,
                              const double *__restrict__ eri, double *__restrict__ eq) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npair * nqp) return;
    const i64 P = i / nqp;
    const int q = (int)(i % nqp);
    eq[i] = q < nq ? eri[tri_idx(P, qpair[q])] : 0.0;
}

int dci_build(sbd_ctx *ctx) {
    DciState &d = ctx->dci;
    if (d.valid) return SBD_OK;
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    const int norb = ctx->norb;
    d.nq = norb * (norb - 1) / 2;
    d.nqp = std::max(8, (d.nq + 7) / 8 * 8);
    std::vector<int32_t> qmap(ctx->npair, 0), qpair(d.nq);
    int q = 0;
    for (int p = 1; p < norb; ++p)
        for (int r = 0; r < p; ++r) {
            qmap[tri_idx(p, r)] = q;
            qpair[q++] = (int32_t)tri_idx(p, r);
        }
    // largest single count per alpha / beta string (host copies of the offsets)
    auto max_count = [&](const Sector &s, int &mx) -> int {
        std::vector<int64_t> off(s.n + 1);
        SBD_CUDA(ctx, cudaMemcpy(off.data(), s.s_off.p, sizeof(int64_t) * (s.n + 1), cudaMemcpyDeviceToHost));
        mx = 0;
        for (i64 i = 0; i < s.n; ++i) mx = std::max(mx, (int)(off[i + 1] - off[i]));
        return SBD_OK;
    };
    int ka = 0, kb = 0;
    int rc = max_count(A, ka);
    if (rc) return rc;
    rc = max_count(B, kb);
    if (rc) return rc;
    d.kp_max = std::max(4, (ka + 3) & ~3);
    d.kb_max = kb;
    d.ld_e = dci_ld_e(d.kp_max);  // = 4 mod 16
    d.nt = kNT;
    d.ntiles = (int)((B.n + kNT - 1) / kNT);
    DevBuf qm, qp;
    SBD_CUDA(ctx, qm.ensure(sizeof(int32_t) * qmap.size()));
    SBD_CUDA(ctx, qp.ensure(sizeof(int32_t) * std::max<size_t>(1, qpair.size())));
    SBD_CUDA(ctx, cudaMemcpy(qm.p, qmap.data(), sizeof(int32_t) * qmap.size(), cudaMemcpyHostToDevice));
    if (d.nq) SBD_CUDA(ctx, cudaMemcpy(qp.p, qpair.data(), sizeof(int32_t) * qpair.size(), cudaMemcpyHostToDevice));
    SBD_CUDA(ctx, d.eq.ensure(sizeof(double) * ctx->npair * d.nqp));
    dci_eq_kernel<<<grid_for(ctx->npair * d.nqp, 256), 256, 0, ctx->stream>>>(ctx->npair, d.nq, d.nqp,
                                                                               qp.as<int32_t>(), ctx->eri.as<double>(),
                                                                               d.eq.as<double>());
    SBD_LAUNCHED(ctx, "dci_eq_kernel");
    if (kb <= kMaxSingles) {
        SBD_CUDA(ctx, d.ent.ensure(sizeof(uint32_t) * std::max<i64>(1, B.ns)));
        SBD_CUDA(ctx, d.toff.ensure(sizeof(int32_t) * B.n * (d.ntiles + 1)));
        dci_lists_kernel<<<grid_for(B.n, 128), 128, 0, ctx->stream>>>(B.n, B.s_off.as<int64_t>(), B.sconn.as<SConn>(),
                                                                      qm.as<int32_t>(), d.nt, d.ntiles, d.ent.as<uint32_t>(),
                                                                      d.toff.as<int32_t>());
        SBD_LAUNCHED(ctx, "dci_lists_kernel");
        // per-tile ELL blocks (coalesced, independent loads in the kernel's gather)
        SBD_CUDA(ctx, d.wt.ensure(sizeof(int32_t) * d.ntiles));
        SBD_CUDA(ctx, cudaMemsetAsync(d.wt.p, 0, sizeof(int32_t) * d.ntiles, ctx->stream));
        dci_width_kernel<<<grid_for(B.n, 128), 128, 0, ctx->stream>>>(B.n, d.toff.as<int32_t>(), d.ntiles,
                                                                      d.wt.as<int32_t>());
        SBD_LAUNCHED(ctx, "dci_width_kernel");
        std::vector<int32_t> wh(d.ntiles);
        SBD_CUDA(ctx, cudaMemcpyAsync(wh.data(), d.wt.p, sizeof(int32_t) * d.ntiles, cudaMemcpyDeviceToHost, ctx->stream));
        SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        std::vector<int64_t> wo(d.ntiles + 1, 0);
        d.wmax = 0;
        for (int t = 0; t < d.ntiles; ++t) {  // blocks start 16-byte aligned (cp.async staging)
            wo[t + 1] = wo[t] + (((i64)wh[t] * B.n + 7) & ~(i64)7);
            d.wmax = std::max(d.wmax, wh[t]);
        }
        SBD_CUDA(ctx, d.woff.ensure(sizeof(int64_t) * (d.ntiles + 1)));
        SBD_CUDA(ctx, cudaMemcpy(d.woff.p, wo.data(), sizeof(int64_t) * (d.ntiles + 1), cudaMemcpyHostToDevice));
        SBD_CUDA(ctx, d.ell.ensure(sizeof(uint16_t) * std::max<i64>(8, wo[d.ntiles])));
        dci_ell_kernel<<<grid_for(B.n, 128), 128, 0, ctx->stream>>>(B.n, d.toff.as<int32_t>(), d.ent.as<uint32_t>(),
                                                                    d.ntiles, d.wt.as<int32_t>(), d.woff.as<int64_t>(),
                                                                    (uint32_t)d.nqp << 1, d.ell.as<uint16_t>());
        SBD_LAUNCHED(ctx, "dci_ell_kernel");
    }
    SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // qm/qp are released on return
    d.valid = true;
    return SBD_OK;
}

template <int MFW, int KS, int PPT>
int launch_dci(sbd_ctx *ctx, const DciArgs &a, size_t smem) {
    SBD_CUDA(ctx, sbd_smem_attr((const void *)cross_kernel_dci<MFW, KS, PPT>, ctx->device, smem));
    cross_kernel_dci<MFW, KS, PPT><<<(unsigned)ctx->num_sms, kDciThreads, smem, ctx->stream>>>(a);
    SBD_LAUNCHED(ctx, "cross_kernel_dci");
    return SBD_OK;
}

template <int MFW, int KS>
int launch_dci_ppt(sbd_ctx *ctx, const DciArgs &a, size_t smem) {
    const i64 ppt = (a.nb + kDciThreads - 1) / kDciThreads;
    if (ppt <= 2) return launch_dci<MFW, KS, 2>(ctx, a, smem);
    if (ppt <= 4) return launch_dci<MFW, KS, 4>(ctx, a, smem);
    return launch_dci<MFW, KS, 8>(ctx, a, smem);
}

// (row fragments per warp, k-steps in registers) instantiated: up to 36 alpha singles per string and
// MFW * KS <= 32 doubles of E per thread (no spills at 512 threads: cfg1 is MFW 3, KS 9)
bool dci_shape(int nqp, int kp, int *mfw, int *ks) {
    *mfw = (nqp / 8 + kMG - 1) / kMG;
    *ks = kp <= 16 ? 4 : 9;
    return kp <= 36 && *mfw <= 4 && *mfw * *ks <= 32;
}

}  // namespace

// Whether the direct-CI task 0 serves this context (SBD_CROSS_DCI=0/1 forces it off / on where it can run).
bool sbd_dci_eligible(sbd_ctx *ctx, const double *x_full) {
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    const char *env = getenv("SBD_CROSS_DCI");
    if (env && env[0] == '0') return false;
    const int norb = ctx->norb, nq = norb * (norb - 1) / 2;
    const int nqp = std::max(8, (nq + 7) / 8 * 8);
    if (nqp > 120 || B.n % 2 != 0 || B.n > (i64)kDciThreads * 8 || B.n * (i64)((B.n + 31) / 32 + 1) >= (1ll << 31) ||
        B.ns >= (1ll << 31) || (reinterpret_cast<uintptr_t>(x_full) & 15) != 0 || A.ns == 0 || B.ns == 0)
        return false;
    const int na = A.n_elec, nbe = B.n_elec;
    if ((i64)na * (norb - na) > 64 || (i64)nbe * (norb - nbe) > kMaxSingles) return false;
    const int kp = std::max(4, (na * (norb - na) + 3) & ~3);
    int mfw, ks;
    if (!dci_shape(nqp, kp, &mfw, &ks) || dci_smem(nqp, kp, dci_ld_e(kp)) > kDciSmemMax) return false;
    if (!(env && env[0] == '1')) {
        // tensor-core FMAs (nqp per beta column) against SELL terms (in-set beta singles per string):
        // the contraction runs ~14x faster per FMA than the gathered terms (cfg1 measurement)
        const double cbar_b = (double)B.ns / (double)std::max<i64>(1, B.n);
        if (8.0 * cbar_b < (double)nqp) return false;
    }
    // the widest tile's gather block must fit next to E, the slab and G (known once the lists exist)
    if (dci_build(ctx) != SBD_OK) return false;
    const DciState &d = ctx->dci;
    return d.kb_max <= kMaxSingles && dci_smem(nqp, kp, dci_ld_e(kp), (i64)d.wmax * B.n) <= kDciSmemMax;
}

int sbd_cross_dci(sbd_ctx *ctx, const double *x_full, double *y, bool additive, const SConn *sconn) {
    int rc = dci_build(ctx);
    if (rc) return rc;
    const DciState &d = ctx->dci;
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    if (d.kb_max > kMaxSingles) return sbd_fail(ctx, SBD_EINVAL, "direct-CI task 0: too many beta singles per string");
    DciArgs a{};
    a.n_rows = ctx->own_rows();
    a.row_base = ctx->own_lo();
    a.nb = B.n;
    a.X = x_full;
    a.Y = y;
    a.a_s_off = A.s_off.as<int64_t>();
    a.a_sconn = sconn ? sconn : A.sconn.as<SConn>();
    a.eq = d.eq.as<double>();
    a.nqp = d.nqp;
    a.kp_max = d.kp_max;
    a.ld_e = d.ld_e;
    a.ell = d.ell.as<uint16_t>();
    a.woff = d.woff.as<int64_t>();
    a.wt = d.wt.as<int32_t>();
    a.ntiles = d.ntiles;
    a.wmax = d.wmax;
    a.add = additive;
    const size_t smem = dci_smem(d.nqp, d.kp_max, d.ld_e, (i64)d.wmax * B.n);
    int mfw, ks;
    if (!dci_shape(d.nqp, d.kp_max, &mfw, &ks) || smem > kDciSmemMax)
        return sbd_fail(ctx, SBD_EINVAL, "direct-CI task 0: shape not served");
    if (ks == 4) {
        if (mfw <= 2) return launch_dci_ppt<2, 4>(ctx, a, smem);
        if (mfw == 3) return launch_dci_ppt<3, 4>(ctx, a, smem);
        return launch_dci_ppt<4, 4>(ctx, a, smem);
    }
    if (mfw <= 2) return launch_dci_ppt<2, 9>(ctx, a, smem);
    return launch_dci_ppt<3, 9>(ctx, a, smem);
}
