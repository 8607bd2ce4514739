// The Davidson sigma build y = H x over the alpha x beta determinant tensor.
//
// Reference: _product_row (apply.py:183-245) evaluates, for each bra row
// (ia, ib), the diagonal, task 1 (beta singles/doubles, alpha fixed), task 2
// (alpha singles/doubles, beta fixed) and task 0 (alpha single x beta single),
// recomputing every Slater-Condon element from determinant words
// (_hij_words, apply.py:152-177).
//
// B200 formulation.  With X the (n_alpha x n_beta) amplitude matrix:
//
//   sigma = diag o X + A X + (B X^T)^T + cross
//
// where A (B) is the alpha (beta) same-spin connection matrix.  A double's
// element is spectator independent (one f64 per CSR entry); a single's is
// phase*(F + J[P][spectator]) with F per entry and J per (orbital pair,
// spectator string) precomputed once (sbd_excite.cu).  Both same-spin parts
// become "row streams": output row r accumulates c_e * X[tgt_e, :] over its
// CSR entries -- 128-bit coalesced loads of whole X rows, no gathers, no
// atomics, every output element owned by one lane.  The beta part runs on
// X^T (one tiled transpose) so it has the same shape; its result Y^T is
// read back, column by column, in the alpha kernel's epilogue.
// Grid order keeps all SMs on one column tile of X at a time, so the ~c-bar
// re-reads of each X row segment are served from L2.
#include <algorithm>
#include <cstdlib>

#include "sbd_internal.cuh"
#include "sbd_ptx.cuh"

namespace {

constexpr int kRowsPerCta = 8;   // one warp per output row
constexpr int kColsPerWarp = 128;  // 4 columns per lane

struct SideArgs {
    i64 n_rows, row_base;          // output rows (local) and global row of local row 0
    i64 n_cols, col_base;          // output columns; J column offset
    const double *X;               // input rows indexed by connection target
    i64 ldx;
    double *Y;
    i64 ldy;
    const int64_t *conn_off;       // indexed by global row
    const Conn *conn;
    const double *J;               // J[P * ldj + col_base + col] of the spectator sector
    i64 ldj;
    // alpha side only
    const double *diag;            // [n_rows][ldy]
    const double *YT;              // beta-side result, [n_cols][ldyt]
    i64 ldyt;
    const int64_t *a_s_off;        // rows with alpha singles carry task 0 in Y (cross_kernel); null: no task 0
    i64 tile0;                     // first column tile (pipelined host path launches tile ranges)
    // Y^T layout.  false: [n_beta][ld_t] (alpha row contiguous).  true (blocked): blocks of 8
    // alpha rows, [ld_t / 8][n_beta][8] -- the alpha CTA's 8 rows x 256 columns are one
    // contiguous 16 KB block instead of 256 scattered 64-byte pieces (L1-friendly reads)
    bool ytb;
    // partitioned passes (DIST kernels, sbd_alpha_pass): local row r streams the connections
    // seg_off[r * seg_stride + seg_lo] .. seg_off[r * seg_stride + seg_hi] of `conn`; its own x
    // row is X[xo_row0 + r]; epi adds diag o x + (B X^T)^T and writes y, acc_in adds onto y
    const int64_t *seg_off;
    i64 seg_stride, xo_row0;
    int seg_lo, seg_hi;
    bool epi, acc_in;
};

template <bool VEC>
__device__ __forceinline__ i64 lane_col(i64 c0, int lane, int j) {
    return VEC ? c0 + (j >> 1) * 64 + 2 * lane + (j & 1) : c0 + j * 32 + lane;
}

template <bool VEC, bool RO = true>
__device__ __forceinline__ void load4(const double *__restrict__ row, i64 c0, int lane, const bool (&ok)[4],
                                      double (&v)[4]) {
    if (VEC) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (ok[2 * h]) {
                const double2 *pp = reinterpret_cast<const double2 *>(row + c0 + h * 64 + 2 * lane);
                double2 t = RO ? __ldg(pp) : *pp;
                v[2 * h] = t.x;
                v[2 * h + 1] = t.y;
            } else {
                v[2 * h] = v[2 * h + 1] = 0.0;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = ok[j] ? (RO ? __ldg(row + c0 + j * 32 + lane) : row[c0 + j * 32 + lane]) : 0.0;
    }
}

template <bool VEC, bool ALPHA, bool DIST = false>
__global__ void __launch_bounds__(kRowsPerCta * 32) side_kernel(SideArgs a) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 r = (i64)blockIdx.x * kRowsPerCta + w;
    const i64 c0 = (i64)blockIdx.y * kColsPerWarp;
    const bool row_ok = r < a.n_rows;
    bool ok[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) ok[j] = lane_col<VEC>(c0, lane, j) < a.n_cols;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};

    if (row_ok) {
        const i64 g = a.row_base + r;
        const i64 e0 = DIST ? a.seg_off[r * a.seg_stride + a.seg_lo] : a.conn_off[g];
        const i64 e1 = DIST ? a.seg_off[r * a.seg_stride + a.seg_hi] : a.conn_off[g + 1];
        i64 e = e0;
        // batches of 4 connections: 8 independent 128-bit loads in flight per lane
        for (; e + 4 <= e1; e += 4) {
            Conn cn[4];
            double xv[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) cn[u] = a.conn[e + u];
#pragma unroll
            for (int u = 0; u < 4; ++u) load4<VEC>(a.X + (i64)cn[u].tgt * a.ldx, c0, lane, ok, xv[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (cn[u].info == 0) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[j] = fma(cn[u].c, xv[u][j], acc[j]);
                } else {
                    const int P = abs(cn[u].info) - 1;
                    const double sg = cn[u].info > 0 ? 1.0 : -1.0;
                    const double *jr = a.J + (i64)P * a.ldj + a.col_base;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        double jv = ok[j] ? __ldg(jr + lane_col<VEC>(c0, lane, j)) : 0.0;
                        acc[j] = fma(fma(sg, jv, cn[u].c), xv[u][j], acc[j]);
                    }
                }
            }
        }
        for (; e < e1; ++e) {
            Conn cn = a.conn[e];
            double xv[4];
            load4<VEC>(a.X + (i64)cn.tgt * a.ldx, c0, lane, ok, xv);
            if (cn.info == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j] = fma(cn.c, xv[j], acc[j]);
            } else {
                const int P = abs(cn.info) - 1;
                const double sg = cn.info > 0 ? 1.0 : -1.0;
                const double *jr = a.J + (i64)P * a.ldj + a.col_base;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    double jv = ok[j] ? __ldg(jr + lane_col<VEC>(c0, lane, j)) : 0.0;
                    acc[j] = fma(fma(sg, jv, cn.c), xv[j], acc[j]);
                }
            }
        }
    }

    if (ALPHA && (!DIST || a.epi)) {  // uniform per launch: every thread reaches the barrier
        // + (B X^T)^T : tile YT[c0:c0+128, r0:r0+8] through shared memory
        __shared__ double tile[kColsPerWarp][kRowsPerCta + 1];
        const i64 r0 = (i64)blockIdx.x * kRowsPerCta;
        {
            const int i = threadIdx.x >> 1, half = (threadIdx.x & 1) * 4;
            if (c0 + i < a.n_cols) {
                const double2 *src = reinterpret_cast<const double2 *>(
                    a.ytb ? a.YT + ((r0 >> 3) * a.n_cols + c0 + i) * 8 + half : a.YT + (c0 + i) * a.ldyt + r0 + half);
                double2 u = src[0], v = src[1];
                tile[i][half + 0] = u.x;
                tile[i][half + 1] = u.y;
                tile[i][half + 2] = v.x;
                tile[i][half + 3] = v.y;
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const i64 lc = lane_col<VEC>(c0, lane, j) - c0;
            if (row_ok && ok[j]) acc[j] += tile[lc][w];
        }
        if (row_ok) {
            const i64 g = a.row_base + r;
            // diagonal term (apply.py:217)
            double dv[4], xo[4];
            load4<VEC>(a.diag + r * a.ldy, c0, lane, ok, dv);
            load4<VEC>(a.X + (DIST ? a.xo_row0 + r : g) * a.ldx, c0, lane, ok, xo);
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = fma(dv[j], xo[j], acc[j]);
            // task 0, already in Y for rows with alpha singles (cross_kernel)
            if (a.a_s_off != nullptr && a.a_s_off[g + 1] != a.a_s_off[g]) {
                double pv[4];
                load4<VEC, false>(a.Y + r * a.ldy, c0, lane, ok, pv);
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j] += pv[j];
            }
        }
    }

    if (DIST && a.acc_in && row_ok) {
        double pv[4];
        load4<VEC, false>(a.Y + r * a.ldy, c0, lane, ok, pv);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += pv[j];
    }
    if (row_ok) {
        double *yr = a.Y + r * a.ldy;
        if (VEC) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const i64 c = c0 + h * 64 + 2 * lane;
                if (ok[2 * h] && ok[2 * h + 1]) {
                    __stcs(reinterpret_cast<double2 *>(yr + c), make_double2(acc[2 * h], acc[2 * h + 1]));
                } else if (ok[2 * h]) {
                    yr[c] = acc[2 * h];
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (ok[j]) yr[c0 + j * 32 + lane] = acc[j];
        }
    }
}

// Asynchronous-copy variant of side_kernel (16-byte aligned rows).  A warp
// owns one output row and a tile of kTW = 256 columns; each lane streams its
// own 8 columns of every connection's x row segment with cp.async (16-byte
// LDGSTS, L1 bypass) into a private ring of kRing shared-memory slots, so
// kRing segments per lane are in flight without holding registers -- the
// register-staged version is latency-bound at ~100 KB in flight per SM.  A
// lane only ever reads back the bytes it copied itself, so cp.async.wait_group
// is the only synchronisation (no barriers in the stream).
constexpr int kTW = 256;

constexpr int kSideCtas = 4;  // resident CTAs per SM: registers <= 64, 4 x 48 KB rings (5 CTAs spill and need a 2-slot ring: slower)

template <bool ALPHA>
struct SideAsync {
    static constexpr int kRing = 3;
    static constexpr size_t smem() { return sizeof(double) * (size_t)kRowsPerCta * kRing * kTW; }
};

template <bool ALPHA, bool DIST = false>
__global__ void __launch_bounds__(kRowsPerCta * 32, kSideCtas) side_kernel_async(SideArgs a) {
    const bool EPI = ALPHA && (!DIST || a.epi);  // uniform per launch
    constexpr int R = SideAsync<ALPHA>::kRing;
    extern __shared__ __align__(128) unsigned char ssm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *ring = reinterpret_cast<double *>(ssm) + (size_t)w * R * kTW;
    const i64 r = (i64)blockIdx.x * kRowsPerCta + w;
    const i64 c0 = ((i64)blockIdx.y + a.tile0) * kTW;
    const i64 ncol = min((i64)kTW, a.n_cols - c0);
    const bool row_ok = r < a.n_rows;
    bool ok[8], pair[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        ok[2 * h] = 2 * lane + 64 * h < ncol;
        ok[2 * h + 1] = 2 * lane + 64 * h + 1 < ncol;
        pair[h] = ok[2 * h];  // rows are padded to even length: the pair is readable
    }
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    i64 nstream = 0;
    if (row_ok) {
        const i64 g = a.row_base + r;
        const i64 own = DIST ? a.xo_row0 + r : g;  // this row's own x row in X
        const i64 e0 = DIST ? a.seg_off[r * a.seg_stride + a.seg_lo] : a.conn_off[g];
        const i64 n = (DIST ? a.seg_off[r * a.seg_stride + a.seg_hi] : a.conn_off[g + 1]) - e0;
        // Alpha side: the two ring slots the stream frees last are refilled with the
        // epilogue's diag and own-x segments (ring positions n and n + 1), so their
        // HBM latency overlaps the stream's tail instead of following it.  The
        // positions >= n are peeled off the hot loop's issue (one uniform branch):
        // same-box A/B -7% at 1e9 dets, -3% at cfg4, neutral at cfg2 (an earlier
        // form that tested every issue for n and n + 1 cost 3-4% there).
        auto issue = [&](i64 i, int slot) {
            if (i < n) {
                const double *src = a.X + (i64)a.conn[e0 + i].tgt * a.ldx + c0;
                double *dst = ring + (size_t)slot * kTW;
#pragma unroll
                for (int h = 0; h < 4; ++h)
                    if (pair[h]) cp_async16(dst + 2 * lane + 64 * h, src + 2 * lane + 64 * h);
            }
            cp_async_commit();
        };
        // the stream's last two issues (positions n, n + 1) carry the epilogue operands
        auto issue_epi = [&](i64 i, int slot) {
            const double *src = i < n ? a.X + (i64)a.conn[e0 + i].tgt * a.ldx + c0
                                      : (i == n ? a.diag + r * a.ldy + c0 : a.X + own * a.ldx + c0);
            if (i <= n + 1) {
                double *dst = ring + (size_t)slot * kTW;
#pragma unroll
                for (int h = 0; h < 4; ++h)
                    if (pair[h]) cp_async16(dst + 2 * lane + 64 * h, src + 2 * lane + 64 * h);
            }
            cp_async_commit();
        };
        if (EPI) nstream = n;
#pragma unroll
        for (int i = 0; i < R - 1; ++i) {
            if (EPI) issue_epi(i, i);
            else issue(i, i);
        }
        int slot = 0;
        for (i64 i = 0; i < n; ++i) {
            const i64 nx = i + R - 1;
            const int ns = slot == 0 ? R - 1 : slot - 1;
            if (EPI && nx >= n) issue_epi(nx, ns);
            else issue(nx, ns);
            const Conn cn = a.conn[e0 + i];
            cp_async_wait<R - 1>();
            const double *src = ring + (size_t)slot * kTW;
            double2 v[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) v[h] = *reinterpret_cast<const double2 *>(src + 2 * lane + 64 * h);
            if (cn.info == 0) {
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    acc[2 * h] = fma(cn.c, v[h].x, acc[2 * h]);
                    acc[2 * h + 1] = fma(cn.c, v[h].y, acc[2 * h + 1]);
                }
            } else {
                const int P = abs(cn.info) - 1;
                const double sg = cn.info > 0 ? 1.0 : -1.0;
                const double *jr = a.J + (i64)P * a.ldj + a.col_base + c0;
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int cc = 2 * lane + 64 * h;
                    const double j0 = ok[2 * h] ? __ldg(jr + cc) : 0.0, j1 = ok[2 * h + 1] ? __ldg(jr + cc + 1) : 0.0;
                    acc[2 * h] = fma(fma(sg, j0, cn.c), v[h].x, acc[2 * h]);
                    acc[2 * h + 1] = fma(fma(sg, j1, cn.c), v[h].y, acc[2 * h + 1]);
                }
            }
            if (++slot == R) slot = 0;
        }
        cp_async_wait<0>();
    }

    if (EPI && row_ok) {
        // + (B X^T)^T: Y^T[c, r] read directly.  The CTA's 8 rows r0..r0+7 are 64
        // contiguous bytes of each Y^T column, so the 8 warps share one L1 line per
        // column and no block barrier (warps finish unevenly) is needed.
        const i64 g = a.row_base + r;
        // diag and own-x segments, staged by the stream's last two issues
        const double *dring = ring + (size_t)(nstream % R) * kTW, *xring = ring + (size_t)((nstream + 1) % R) * kTW;
        const bool t0 = a.a_s_off != nullptr && a.a_s_off[g + 1] != a.a_s_off[g];
        const double *yrow = a.Y + r * a.ldy + c0;
        // Y^T[c0 + cc][r] = ytc[cc * yts]
        const double *ytc = a.ytb ? a.YT + ((r >> 3) * a.n_cols + c0) * 8 + (r & 7) : a.YT + c0 * a.ldyt + r;
        const i64 yts = a.ytb ? 8 : a.ldyt;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int cc = 2 * lane + 64 * h;
            if (ok[2 * h + 1]) {
                const double2 d = *reinterpret_cast<const double2 *>(dring + cc);
                const double2 x = *reinterpret_cast<const double2 *>(xring + cc);
                const double t0v = __ldg(ytc + cc * yts), t1v = __ldg(ytc + (cc + 1) * yts);
                acc[2 * h] = fma(d.x, x.x, acc[2 * h] + t0v);
                acc[2 * h + 1] = fma(d.y, x.y, acc[2 * h + 1] + t1v);
                if (t0) {
                    const double2 p = *reinterpret_cast<const double2 *>(yrow + cc);
                    acc[2 * h] += p.x;
                    acc[2 * h + 1] += p.y;
                }
            } else if (ok[2 * h]) {
                acc[2 * h] = fma(dring[cc], xring[cc], acc[2 * h] + __ldg(ytc + cc * yts));
                if (t0) acc[2 * h] += yrow[cc];
            }
        }
    }

    if (DIST && a.acc_in && row_ok) {  // later pass of the partitioned sigma: add onto y
        const double *yrow = a.Y + r * a.ldy + c0;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int cc = 2 * lane + 64 * h;
            if (ok[2 * h + 1]) {
                const double2 p = __ldcs(reinterpret_cast<const double2 *>(yrow + cc));
                acc[2 * h] += p.x;
                acc[2 * h + 1] += p.y;
            } else if (ok[2 * h]) {
                acc[2 * h] += yrow[cc];
            }
        }
    }
    if (row_ok) {
        if (!ALPHA && a.ytb) {  // blocked Y^T: element (r, c) at ((c >> 3) * n_rows + r) * 8 + (c & 7)
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const i64 c = c0 + 2 * lane + 64 * h;
                double *p = a.Y + ((c >> 3) * a.n_rows + r) * 8 + (c & 7);
                if (ok[2 * h + 1]) __stcs(reinterpret_cast<double2 *>(p), make_double2(acc[2 * h], acc[2 * h + 1]));
                else if (ok[2 * h]) *p = acc[2 * h];
            }
        } else {
            double *yr = a.Y + r * a.ldy + c0;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int cc = 2 * lane + 64 * h;
                if (ok[2 * h + 1]) __stcs(reinterpret_cast<double2 *>(yr + cc), make_double2(acc[2 * h], acc[2 * h + 1]));
                else if (ok[2 * h]) yr[cc] = acc[2 * h];
            }
        }
    }
}

// Task 0, the alpha-single x beta-single opposite-spin doubles (apply.py:235-238):
//   Y[r, ib] = sum_{k in aS(g)} s_k sum_{m in bS(ib)} s_m (Pa_k | Pb_m) X[ja_k, jb_m]
// written for rows that have alpha singles (the streaming kernel adds it).
//
// Work list: the flat list of alpha-single entries of the owned rows, split
// over CTAs at row boundaries, so a row's entries stay in one CTA.  The beta
// singles are a chunked sliced ELL (sbd_excite.cu build_sell): beta strings
// sorted by single count into groups of 32 positions; per chunk of targets
// each group is slot-major and padded to its widest position with entries
// that read a zero slot.  Lane l of warp w owns position l of groups
// w + 32 j (j < CPT) and keeps their sums in registers across all entries of
// a row; the row is written once (no atomics, no read-back).  An entry packs
// the chunk-local target and the column of a sign-folded ERI row, so the
// inner loop is: shared load, shift, mask, two shared gathers, one FMA.
//
// Staged variant: per (entry, chunk) item, the x row chunk ja_k[h*C, h*C+C)
// and the ERI row (Pa_k, s_k) are TMA bulk-copied (cp.async.bulk + mbarrier)
// into one of two shared-memory stages; full[s] counts the bytes, empty[s]
// counts warps done with it, so a fast warp runs ahead into the other stage
// and thread 0 refills a stage as soon as every warp released it.  The SELL
// itself is also resident in shared memory when it fits.
constexpr int kCrossThreads = 1024;      // staged: one CTA per SM
constexpr int kCrossThreadsFlat = 256;   // flat: group tiles x entry ranges

__device__ __forceinline__ i64 snap_entry(i64 t, i64 e_end, const int64_t *__restrict__ a_s_off,
                                          const int32_t *__restrict__ a_row) {
    if (t >= e_end) return e_end;
    const i64 g = a_row[t];
    return t == a_s_off[g] ? t : a_s_off[g + 1];
}

struct CrossArgs {
    i64 n_rows, row_base, nb;
    const double *X;
    double *Y;
    const int64_t *a_s_off;
    const SConn *a_sconn;
    const int32_t *a_row;
    const int32_t *goff;     // beta SELL group offsets [H][groups+1]
    const int32_t *col;      // beta SELL position -> beta string
    const uint32_t *ent;     // beta SELL entries
    i64 groups, H, chunk;
    int pbits;
    const double *vsg;       // sign-folded ERI rows, row (P, s) at (2P + s) * 2 ld
    i64 ld;
    i64 gz;                  // groups processed (a prefix: groups are sorted by single count)
    bool add;                // y += task 0 on the processed positions (run after the alpha side)
};

__device__ __forceinline__ const double *vrow(const CrossArgs &a, const SConn &sa) {
    return a.vsg + (i64)(2 * (abs(sa.info) - 1) + (sa.info < 0)) * 2 * a.ld;
}

// acc[j] += sum over the item's entries of position (g_lo + warp + j*nw, lane)
template <int CPT, bool CHECK>
__device__ __forceinline__ void cross_accumulate(double (&acc)[CPT], const CrossArgs &a, const int32_t *goff_h,
                                                 const uint32_t *ent, const double *xr, const double *vr, i64 g_lo,
                                                 int nw) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t pmask = (1u << a.pbits) - 1u, nul = (uint32_t)a.chunk;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        const i64 g = g_lo + warp + (i64)j * nw;
        if (g < a.gz) {
            const int o0 = goff_h[g], w = (goff_h[g + 1] - o0) >> 5;
            const uint32_t *ep = ent + o0 + lane;
            int q = 0;
            for (; q + 2 <= w; q += 2) {
                const uint32_t p0 = ep[32 * q], p1 = ep[32 * q + 32];
                if (CHECK) {
                    if ((p0 >> a.pbits) != nul) acc[j] = fma(vr[p0 & pmask], xr[p0 >> a.pbits], acc[j]);
                    if ((p1 >> a.pbits) != nul) acc[j] = fma(vr[p1 & pmask], xr[p1 >> a.pbits], acc[j]);
                } else {
                    const double t0 = vr[p0 & pmask] * xr[p0 >> a.pbits];
                    acc[j] = fma(vr[p1 & pmask], xr[p1 >> a.pbits], acc[j] + t0);
                }
            }
            if (q < w) {
                const uint32_t p0 = ep[32 * q];
                if (!CHECK || (p0 >> a.pbits) != nul) acc[j] = fma(vr[p0 & pmask], xr[p0 >> a.pbits], acc[j]);
            }
        }
    }
}

template <int CPT>
__device__ __forceinline__ void cross_store(double (&acc)[CPT], const CrossArgs &a, double *yr, i64 g_lo, int nw) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int c[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {  // all column loads first: one round trip, not CPT
        const i64 g = g_lo + warp + (i64)j * nw;
        c[j] = g < a.gz ? __ldg(a.col + g * 32 + lane) : -1;
    }
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        if (c[j] >= 0) {
            if (a.add) yr[c[j]] += acc[j];
            else yr[c[j]] = acc[j];
        }
        acc[j] = 0.0;
    }
}

__host__ __device__ inline i64 cross_stage_doubles(i64 chunk, i64 ld) { return chunk + 2 + 2 * ld; }
constexpr int kCrossStages = 3;


// Warp-specialised pipeline: the last warp produces (TMA into kCrossStages
// stages, L2 prefetch two items further ahead), the other warps consume.
template <int CPT, bool SENT>
__global__ void __launch_bounds__(kCrossThreads, 1) cross_kernel_tma(CrossArgs a) {
    extern __shared__ __align__(128) unsigned char csm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(csm);
    uint64_t *empty = full + kCrossStages;
    double *st0 = reinterpret_cast<double *>(csm + 128);
    const i64 sdbl = cross_stage_doubles(a.chunk, a.ld);
    int32_t *sgoff = reinterpret_cast<int32_t *>(st0 + kCrossStages * sdbl);
    const i64 ngoff = a.H * (a.groups + 1);
    uint32_t *sent = reinterpret_cast<uint32_t *>(sgoff + ((ngoff + 3) & ~(i64)3));
    constexpr int kC = kCrossThreads / 32 - 1;  // consumer warps
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 E0 = a.a_s_off[a.row_base], E1 = a.a_s_off[a.row_base + a.n_rows];
    const i64 tot = E1 - E0;
    const i64 e0 = snap_entry(E0 + tot * blockIdx.x / gridDim.x, E1, a.a_s_off, a.a_row);
    const i64 e1 = snap_entry(E0 + tot * (blockIdx.x + 1) / gridDim.x, E1, a.a_s_off, a.a_row);
    if (e0 >= e1) return;
    const i64 nitems = (e1 - e0) * a.H;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kCrossStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kC);
        }
        mbar_fence_init();
    }
    if (threadIdx.x < kCrossStages) {  // zero slots read by padding entries
        st0[threadIdx.x * sdbl + a.chunk] = 0.0;
        st0[threadIdx.x * sdbl + a.chunk + 1] = 0.0;
    }
    for (i64 i = threadIdx.x; i < ngoff; i += kCrossThreads) sgoff[i] = a.goff[i];
    if (SENT) {
        const i64 nent = a.goff[ngoff - 1];
        for (i64 i = threadIdx.x; i < nent / 4; i += kCrossThreads)
            reinterpret_cast<uint4 *>(sent)[i] = __ldg(reinterpret_cast<const uint4 *>(a.ent) + i);
        for (i64 i = (nent & ~(i64)3) + threadIdx.x; i < nent; i += kCrossThreads) sent[i] = a.ent[i];
    }
    __syncthreads();
    if (warp == kC) {
        if (lane != 0) return;
        const uint32_t bv = (uint32_t)(2 * a.ld * sizeof(double));
        i64 e = e0, h = 0, pe = e0, ph_ = 0;  // item being issued; item being prefetched
        auto advance = [&](i64 &ee, i64 &hh) {
            if (++hh == a.H) { hh = 0; ++ee; }
        };
        for (int k = 0; k < 2 && pe < e1; ++k) {  // prefetch window
            prefetch_l2(a.X + (i64)a.a_sconn[pe].tgt * a.nb + ph_ * a.chunk,
                        (uint32_t)(min(a.chunk, a.nb - ph_ * a.chunk) * sizeof(double)));
            advance(pe, ph_);
        }
        for (i64 item = 0; item < nitems; ++item) {
            const int s = (int)(item % kCrossStages);
            if (item >= kCrossStages) {
                mbar_wait(&empty[s], (uint32_t)(((item / kCrossStages) - 1) & 1));
                fence_proxy_async_smem();  // consumers' generic-proxy reads before the async-proxy refill
            }
            const SConn sa = a.a_sconn[e];
            const i64 c0 = h * a.chunk, cols = min(a.chunk, a.nb - c0);
            double *dst = st0 + s * sdbl;
            const uint32_t bx = (uint32_t)(cols * sizeof(double));
            mbar_arrive_expect_tx(&full[s], bx + bv);
            tma_load_1d(dst, a.X + (i64)sa.tgt * a.nb + c0, bx, &full[s]);
            tma_load_1d(dst + a.chunk + 2, vrow(a, sa), bv, &full[s]);
            advance(e, h);
            if (pe < e1) {
                prefetch_l2(a.X + (i64)a.a_sconn[pe].tgt * a.nb + ph_ * a.chunk,
                            (uint32_t)(min(a.chunk, a.nb - ph_ * a.chunk) * sizeof(double)));
                advance(pe, ph_);
            }
        }
        return;
    }
    double acc[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) acc[j] = 0.0;
    i64 e = e0, h = 0;
    int s = 0;
    uint32_t ph = 0;
    for (i64 item = 0; item < nitems; ++item) {
        mbar_wait(&full[s], ph);
        const double *xr = st0 + s * sdbl;
        cross_accumulate<CPT, false>(acc, a, sgoff + h * (a.groups + 1), SENT ? sent : a.ent, xr, xr + a.chunk + 2, 0,
                                     kC);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == kCrossStages) { s = 0; ph ^= 1u; }
        if (++h == a.H) {
            h = 0;
            const i64 g = a.a_row[e];
            if (e + 1 == e1 || a.a_row[e + 1] != g) cross_store<CPT>(acc, a, a.Y + (g - a.row_base) * a.nb, 0, kC);
            ++e;
        }
    }
}

// Cluster variant (H = 1, whole x rows): a pair of CTAs on two SMs shares
// every entry's x row and ERI row through one TMA multicast (one L2/HBM read
// feeds both shared memories); CTA rank r owns the SELL groups g = 2 gl + r,
// so each CTA keeps only half of the SELL resident and each lane half as
// many accumulators.  Stage release spans the pair: rank 1's producer arms
// its own full barrier and then arrives on rank 0's `peer` barrier; rank 0's
// producer issues the multicast once both CTAs released the stage.
constexpr int kMcStages = 2;
constexpr int kMcPrefetch = 2;

__host__ __device__ inline i64 mc_local_groups(i64 groups, int rank) { return (groups - rank + 1) / 2; }

template <int CPT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kCrossThreads, 1) cross_kernel_mc(CrossArgs a) {
    extern __shared__ __align__(128) unsigned char csm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(csm);
    uint64_t *empty = full + kMcStages;
    uint64_t *peer = empty + kMcStages;
    double *st0 = reinterpret_cast<double *>(csm + 128);
    const i64 sdbl = cross_stage_doubles(a.chunk, a.ld);
    const int rank = (int)cluster_ctarank();
    const i64 ngl = mc_local_groups(a.groups, rank);
    int32_t *lgoff = reinterpret_cast<int32_t *>(st0 + kMcStages * sdbl);
    uint32_t *sent = reinterpret_cast<uint32_t *>(lgoff + ((ngl + 4) & ~(i64)3));
    constexpr int kC = kCrossThreads / 32 - 1;  // consumer warps
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i64 cl = blockIdx.x / 2, ncl = gridDim.x / 2;
    const i64 E0 = a.a_s_off[a.row_base], E1 = a.a_s_off[a.row_base + a.n_rows];
    const i64 tot = E1 - E0;
    const i64 e0 = snap_entry(E0 + tot * cl / ncl, E1, a.a_s_off, a.a_row);
    const i64 e1 = snap_entry(E0 + tot * (cl + 1) / ncl, E1, a.a_s_off, a.a_row);
    const i64 nitems = e1 - e0;  // both CTAs of the pair see the same range
    if (threadIdx.x == 0) {
        for (int i = 0; i < kMcStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kC);
            mbar_init(&peer[i], 1);
        }
        mbar_fence_init();
        // local group offsets (prefix over this rank's groups)
        int32_t o = 0;
        for (i64 gl = 0; gl < ngl; ++gl) {
            const i64 g = 2 * gl + rank;
            lgoff[gl] = o;
            o += a.goff[g + 1] - a.goff[g];
        }
        lgoff[ngl] = o;
    }
    if (threadIdx.x < kMcStages) {  // zero slots read by padding entries
        st0[threadIdx.x * sdbl + a.chunk] = 0.0;
        st0[threadIdx.x * sdbl + a.chunk + 1] = 0.0;
    }
    __syncthreads();
    for (i64 gl = warp; gl < ngl; gl += kCrossThreads / 32) {  // this rank's SELL into shared memory
        const i64 g = 2 * gl + rank;
        const int src = a.goff[g], cnt = a.goff[g + 1] - src, dst = lgoff[gl];
        for (int i = lane; i < cnt; i += 32) sent[dst + i] = __ldg(a.ent + src + i);
    }
    cluster_sync_all();  // barriers of both CTAs initialised before any remote traffic
    if (warp == kC) {
        if (lane == 0 && nitems > 0) {
            const uint32_t bv = (uint32_t)(2 * a.ld * sizeof(double));
            const uint32_t bx = (uint32_t)(a.nb * sizeof(double));
            const uint32_t peer_other = cluster_map(&peer[0], (uint32_t)(rank ^ 1));
            // each rank multicasts half of the row (rank 0 also the ERI row), so both
            // CTAs' TMA units work on every item
            const i64 half = (a.nb / 2 + 1) & ~(i64)1;
            const i64 x0 = rank == 0 ? 0 : half, xn = rank == 0 ? half : a.nb - half;
            for (i64 item = 0; item < nitems; ++item) {
                const int s = (int)(item & 1);
                const uint32_t use = (uint32_t)(item >> 1);
                if (item >= kMcStages) mbar_wait(&empty[s], (use - 1) & 1);  // my consumers released s
                mbar_arrive_expect_tx(&full[s], bx + bv);                       // armed for the whole item
                mbar_arrive_remote(peer_other + (uint32_t)(s * sizeof(uint64_t)));  // my side free + armed
                mbar_wait_cluster(&peer[s], use & 1);                           // the peer's side too
                fence_proxy_async_smem();  // generic-proxy reads of the stage before the async-proxy refill
                const SConn sa = a.a_sconn[e0 + item];
                const double *row = a.X + (i64)sa.tgt * a.nb;
                if (item + kMcPrefetch < nitems && xn > 0)  // next-but-one rows: L2 hits for the TMA
                    prefetch_l2(a.X + (i64)a.a_sconn[e0 + item + kMcPrefetch].tgt * a.nb + x0,
                                (uint32_t)(xn * sizeof(double)));
                double *dst = st0 + s * sdbl;
                if (xn > 0) tma_load_1d_multicast(dst + x0, row + x0, (uint32_t)(xn * sizeof(double)), &full[s], 0x3);
                if (rank == 0) tma_load_1d_multicast(dst + a.chunk + 2, vrow(a, sa), bv, &full[s], 0x3);
            }
        }
    } else {
        // per-group slot ranges never change across items: keep them in registers
        uint32_t gptr[CPT];  // index (in sent) of slot 0 of this lane in group j
        int gw[CPT];         // slots in group j (warp-uniform)
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const i64 gl = warp + (i64)j * kC;
            gw[j] = gl < ngl ? (lgoff[gl + 1] - lgoff[gl]) >> 5 : 0;
            gptr[j] = (uint32_t)(gl < ngl ? lgoff[gl] : 0) + lane;
        }
        const uint32_t pmask = (1u << a.pbits) - 1u, pb = (uint32_t)a.pbits;
        double acc[CPT];
#pragma unroll
        for (int j = 0; j < CPT; ++j) acc[j] = 0.0;
        for (i64 item = 0; item < nitems; ++item) {
            const int s = (int)(item & 1);
            mbar_wait(&full[s], (uint32_t)((item >> 1) & 1));
            const uint32_t xa = smem_u32(st0 + s * sdbl), va = xa + (uint32_t)((a.chunk + 2) * sizeof(double));
            auto term = [&](uint32_t e) {
                return lds_f64(va + ((e & pmask) << 3)) * lds_f64(xa + ((e >> pb) << 3));
            };
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                const int w = gw[j];
                if (w > 0) {
                    const uint32_t ep = smem_u32(sent + gptr[j]);
                    double t = term(lds_u32(ep));
                    if (w > 1) t += term(lds_u32(ep + 128));
                    if (w > 2) {
                        t += term(lds_u32(ep + 256));
                        for (int q = 3; q < w; ++q) t += term(lds_u32(ep + 128 * q));
                    }
                    acc[j] += t;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            const i64 e = e0 + item, g = a.a_row[e];
            if (e + 1 == e1 || a.a_row[e + 1] != g) {
                double *yr = a.Y + (g - a.row_base) * a.nb;
                int c[CPT];
#pragma unroll
                for (int j = 0; j < CPT; ++j) {
                    const i64 gl = warp + (i64)j * kC;
                    c[j] = gl < ngl ? __ldg(a.col + (2 * gl + rank) * 32 + lane) : -1;
                }
#pragma unroll
                for (int j = 0; j < CPT; ++j) {
                    if (c[j] >= 0) {
                        if (a.add) yr[c[j]] += acc[j];
                        else yr[c[j]] = acc[j];
                    }
                    acc[j] = 0.0;
                }
            }
        }
    }
    cluster_sync_all();  // no CTA leaves while its pair may still signal it
}

// Flat (x rows not 16-byte aligned, or too many groups for one CTA):
// grid.x = entry ranges, grid.y = tiles of (warps * CPT) groups; gathers and
// the SELL go through L1/L2.
template <int CPT>
__global__ void __launch_bounds__(kCrossThreadsFlat) cross_kernel_flat(CrossArgs a) {
    constexpr int kW = kCrossThreadsFlat / 32;
    const i64 g_lo = (i64)blockIdx.y * kW * CPT;
    const i64 E0 = a.a_s_off[a.row_base], E1 = a.a_s_off[a.row_base + a.n_rows];
    const i64 tot = E1 - E0;
    const i64 e0 = snap_entry(E0 + tot * blockIdx.x / gridDim.x, E1, a.a_s_off, a.a_row);
    const i64 e1 = snap_entry(E0 + tot * (blockIdx.x + 1) / gridDim.x, E1, a.a_s_off, a.a_row);
    double acc[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) acc[j] = 0.0;
    for (i64 e = e0; e < e1; ++e) {
        const SConn sa = a.a_sconn[e];
        const i64 g = a.a_row[e];
        for (i64 h = 0; h < a.H; ++h)
            cross_accumulate<CPT, true>(acc, a, a.goff + h * (a.groups + 1), a.ent, a.X + (i64)sa.tgt * a.nb + h * a.chunk,
                                        vrow(a, sa), g_lo, kW);
        if (e + 1 == e1 || a.a_row[e + 1] != g) cross_store<CPT>(acc, a, a.Y + (g - a.row_base) * a.nb, g_lo, kW);
    }
}

// X_own [rows][ld_in] -> XT [cols][ld_out]
__global__ void transpose_kernel(const double *__restrict__ in, i64 rows, i64 cols, i64 ld_in, double *__restrict__ out,
                                 i64 ld_out) {
    __shared__ double t[32][33];
    const i64 bc = (i64)blockIdx.x * 32, br = (i64)blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        i64 rr = br + k, cc = bc + threadIdx.x;
        t[k][threadIdx.x] = (rr < rows && cc < cols) ? __ldcs(in + rr * ld_in + cc) : 0.0;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        i64 cc = bc + k, rr = br + threadIdx.x;
        if (cc < cols && rr < rows) out[cc * ld_out + rr] = t[threadIdx.x][k];
    }
}

// Diagonal, reference operation order (apply.py:100-112):
//   e = (e_core + E_a) + E_b; for p in alpha: for q in beta: e += (pp|qq)
__global__ void diag_kernel(i64 n_rows, i64 row_base, i64 nb, const u64 *__restrict__ astr,
                            const u64 *__restrict__ bstr, const double *__restrict__ ea,
                            const double *__restrict__ eb, const double *__restrict__ dpq, int norb, double e_core,
                            double *__restrict__ out) {
    extern __shared__ double sd[];
    for (int i = threadIdx.x; i < norb * norb; i += blockDim.x) sd[i] = dpq[i];
    __syncthreads();
    const i64 total = n_rows * nb;
    for (i64 idx = (i64)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (i64)gridDim.x * blockDim.x) {
        const i64 r = idx / nb, ib = idx - r * nb;
        const i64 g = row_base + r;
        const u64 aw = astr[g], bw = bstr[ib];
        double e = __dadd_rn(__dadd_rn(e_core, ea[g]), eb[ib]);
        for (u64 ta = aw; ta; ta &= ta - 1) {
            const int p = __ffsll((long long)ta) - 1;
            for (u64 tb = bw; tb; tb &= tb - 1) e = __dadd_rn(e, sd[p * norb + __ffsll((long long)tb) - 1]);
        }
        out[idx] = e;
    }
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

bool yt_blocked_enabled() {  // SBD_YT_BLOCKED=0 keeps the row-contiguous Y^T layout (A/B)
    const char *e = getenv("SBD_YT_BLOCKED");
    return !(e && e[0] == '0');
}

i64 sigma_host_chunks() {  // alpha-row chunks of the pipelined host-buffer sigma (SBD_HOST_CHUNKS, A/B)
    const char *e = getenv("SBD_HOST_CHUNKS");
    const long v = e ? strtol(e, nullptr, 10) : 0;
    return v > 0 ? (i64)v : 24;  // 512-row chunks at cfg2: 29.6 vs 29.9 ms with 8 (profiles/r3c, r3d)
}

bool use_side_tma() {  // SBD_SIDE_LDG=1 selects the register-staged stream (A/B measurements)
    const char *e = getenv("SBD_SIDE_LDG");
    return !(e && e[0] == '1');
}

int require_ready(sbd_ctx *ctx) {
    if (!ctx->sec[0].built || !ctx->sec[1].built || (ctx->explicit_mode && !ctx->explicit_built))
        return sbd_fail(ctx, SBD_EINVAL, "tables not built (call sbd_build_tables)");
    return SBD_OK;
}

int require_product(sbd_ctx *ctx) {
    if (ctx->explicit_mode) return sbd_fail(ctx, SBD_EINVAL, "this entry point serves product-mode bases only");
    return SBD_OK;
}

int ensure_diag(sbd_ctx *ctx) {
    if (ctx->diag_valid) return SBD_OK;
    if (ctx->explicit_mode) {
        SBD_CUDA(ctx, ctx->diag.ensure(sizeof(double) * (ctx->n_det + 2)));
        int rc = sbd_explicit_diag(ctx, ctx->diag.as<double>());
        if (rc) return rc;
        ctx->diag_valid = true;
        return SBD_OK;
    }
    const i64 rows = ctx->own_rows(), nb = ctx->sec[1].n;
    SBD_CUDA(ctx, ctx->diag.ensure(sizeof(double) * (rows * nb + 2)));
    if (rows * nb > 0) {
        size_t smem = sizeof(double) * ctx->norb * ctx->norb;
        unsigned blocks = (unsigned)std::min<i64>(grid_for(rows * nb, 256), (i64)ctx->num_sms * 16);
        diag_kernel<<<blocks, 256, smem, ctx->stream>>>(rows, ctx->own_lo(), nb, ctx->sec[0].str.as<u64>(),
                                                        ctx->sec[1].str.as<u64>(), ctx->sec[0].energy.as<double>(),
                                                        ctx->sec[1].energy.as<double>(), ctx->dpq.as<double>(),
                                                        ctx->norb, ctx->e_core, ctx->diag.as<double>());
        SBD_LAUNCHED(ctx, "diag_kernel");
    }
    ctx->diag_valid = true;
    return SBD_OK;
}

int ensure_scratch(sbd_ctx *ctx) {
    const i64 rows = ctx->own_rows(), nb = ctx->sec[1].n;
    ctx->ld_t = std::max<i64>(kColsPerWarp, (rows + kColsPerWarp - 1) / kColsPerWarp * kColsPerWarp);
    size_t bytes = sizeof(double) * (size_t)std::max<i64>(nb, 1) * ctx->ld_t;
    SBD_CUDA(ctx, ctx->xt.ensure(bytes));
    SBD_CUDA(ctx, ctx->yt.ensure(bytes));
    return SBD_OK;
}

template <int CPT, bool SENT>
int launch_cross_tma(sbd_ctx *ctx, const CrossArgs &ca, size_t smem) {
    SBD_CUDA(ctx, sbd_smem_attr((const void *)cross_kernel_tma<CPT, SENT>, ctx->device, smem));
    cross_kernel_tma<CPT, SENT><<<(unsigned)ctx->num_sms, kCrossThreads, smem, ctx->stream>>>(ca);
    SBD_LAUNCHED(ctx, "cross_kernel_tma");
    return SBD_OK;
}

template <int CPT>
int launch_cross_mc(sbd_ctx *ctx, const CrossArgs &ca, size_t smem) {
    SBD_CUDA(ctx, sbd_smem_attr((const void *)cross_kernel_mc<CPT>, ctx->device, smem));
    cross_kernel_mc<CPT><<<(unsigned)ctx->num_sms, kCrossThreads, smem, ctx->stream>>>(ca);
    SBD_LAUNCHED(ctx, "cross_kernel_mc");
    return SBD_OK;
}

template <bool SENT>
int launch_cross_tma_cpt(sbd_ctx *ctx, const CrossArgs &ca, size_t smem, i64 cpt) {
    if (cpt <= 2) return launch_cross_tma<2, SENT>(ctx, ca, smem);
    if (cpt <= 4) return launch_cross_tma<4, SENT>(ctx, ca, smem);
    if (cpt <= 8) return launch_cross_tma<8, SENT>(ctx, ca, smem);
    if (cpt <= 10) return launch_cross_tma<10, SENT>(ctx, ca, smem);
    if (cpt <= 12) return launch_cross_tma<12, SENT>(ctx, ca, smem);
    return launch_cross_tma<14, SENT>(ctx, ca, smem);
}

// Beta SELL groups that hold any single (a prefix: sorted by total count).
i64 sell_nonzero_groups(const Sector &B) {
    const i64 G = B.sell_groups;
    i64 nz = 0;
    for (i64 g = 0; g < G; ++g) {
        i64 w = 0;
        for (i64 h = 0; h < B.sell_h; ++h) w += B.sell_goff_host[h * (G + 1) + g + 1] - B.sell_goff_host[h * (G + 1) + g];
        if (w > 0) nz = g + 1;
    }
    return nz;
}

// Additive task 0: when most beta strings have no in-set single (sparse configs),
// task 0 is added to the finished rows on the few positions it touches, after
// the alpha side, instead of writing whole rows that the alpha side reads back.
bool cross_additive(const sbd_ctx *ctx) {
    const Sector &B = ctx->sec[1];
    const char *e = getenv("SBD_CROSS_ADD");  // 0/1 forces the task-0 order (A/B measurements, tests)
    if (e && *e) return e[0] == '1';
    return B.sell_groups > 0 && 2 * sell_nonzero_groups(B) < B.sell_groups;
}

// Task 0 for the owned rows [r0, r1) (r1 < 0: all of them); y points at owned row 0.
int launch_cross(sbd_ctx *ctx, const double *x_full, double *y, bool additive = false,
                 const SConn *sconn = nullptr, i64 r0 = 0, i64 r1 = -1) {
    if (r1 < 0) r1 = ctx->own_rows();
    if (r0 == 0 && r1 == ctx->own_rows() && sbd_dci_eligible(ctx, x_full)) {
        ctx->last_task0 = 4;
        return sbd_cross_dci(ctx, x_full, y, additive, sconn);
    }
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    CrossArgs ca{};
    ca.n_rows = r1 - r0;
    ca.row_base = ctx->own_lo() + r0;
    ca.nb = B.n;
    ca.X = x_full;
    ca.Y = y + r0 * B.n;
    ca.a_s_off = A.s_off.as<int64_t>();
    ca.a_sconn = sconn ? sconn : A.sconn.as<SConn>();
    ca.a_row = A.s_row.as<int32_t>();
    ca.goff = B.sell_goff.as<int32_t>();
    ca.col = B.sell_col.as<int32_t>();
    ca.ent = B.sell_ent.as<uint32_t>();
    ca.groups = B.sell_groups;
    ca.H = B.sell_h;
    ca.chunk = B.sell_chunk;
    ca.pbits = B.sell_pbits;
    ca.vsg = ctx->vpp.as<double>();
    ca.ld = ctx->ld_vpp;
    ca.gz = ca.groups;
    ca.add = false;
    constexpr size_t kSmemMax = 227 * 1024;
    const i64 ngoff = ca.H * (ca.groups + 1);
    const size_t base = 128 + sizeof(double) * kCrossStages * (size_t)cross_stage_doubles(ca.chunk, ca.ld) +
                        sizeof(int32_t) * (size_t)((ngoff + 3) & ~(i64)3);
    const size_t with_ent = base + sizeof(uint32_t) * (size_t)B.sell_nent;
    const i64 cpt = (ca.groups + kCrossThreads / 32 - 2) / (kCrossThreads / 32 - 1);
    const char *force = getenv("SBD_CROSS_UNSTAGED");  // test knob: exercise the flat variant
    const char *nomc = getenv("SBD_CROSS_NO_CLUSTER");  // test knob: exercise the single-CTA pipeline
    if (additive) {
        ca.gz = sell_nonzero_groups(B);
        ca.add = true;
    }
    if (!(force && force[0] == '1') && !(nomc && nomc[0] == '1') && ca.H == 1 && (B.n % 2 == 0) &&
        aligned16(x_full) && (ctx->num_sms % 2 == 0)) {
        const i64 ngl = mc_local_groups(ca.groups, 0);
        i64 ent0 = 0, ent1 = 0;  // SELL entries per rank (host copy of the offsets)
        for (i64 g = 0; g < ca.groups; ++g) (g % 2 ? ent1 : ent0) += B.sell_goff_host[g + 1] - B.sell_goff_host[g];
        const size_t smem_mc = 128 + sizeof(double) * kMcStages * (size_t)cross_stage_doubles(ca.chunk, ca.ld) +
                               sizeof(int32_t) * (size_t)((ngl + 4) & ~(i64)3) +
                               sizeof(uint32_t) * (size_t)std::max(ent0, ent1);
        const i64 cpt_mc = (ngl + kCrossThreads / 32 - 2) / (kCrossThreads / 32 - 1);
        if (smem_mc <= kSmemMax && cpt_mc <= 8) {
            ctx->last_task0 = 1;
            if (cpt_mc <= 2) return launch_cross_mc<2>(ctx, ca, smem_mc);
            if (cpt_mc <= 4) return launch_cross_mc<4>(ctx, ca, smem_mc);
            if (cpt_mc <= 6) return launch_cross_mc<6>(ctx, ca, smem_mc);
            return launch_cross_mc<8>(ctx, ca, smem_mc);
        }
    }
    const bool staged_ok = !(force && force[0] == '1') && (B.n % 2 == 0) && aligned16(x_full) && cpt <= 14;
    if (staged_ok && (with_ent <= kSmemMax || base <= kSmemMax)) {
        ctx->last_task0 = 2;
        if (with_ent <= kSmemMax) return launch_cross_tma_cpt<true>(ctx, ca, with_ent, cpt);
        return launch_cross_tma_cpt<false>(ctx, ca, base, cpt);
    }
    ctx->last_task0 = 3;
    constexpr int kCpt = 8;
    const i64 gpt = (i64)(kCrossThreadsFlat / 32) * kCpt;
    const i64 tiles = std::max<i64>(1, (ca.gz + gpt - 1) / gpt);
    const unsigned gx = (unsigned)std::max<i64>(1, std::min<i64>((i64)ctx->num_sms * 8 / tiles + 1, ctx->own_rows()));
    dim3 grid(gx, (unsigned)tiles);
    cross_kernel_flat<kCpt><<<grid, kCrossThreadsFlat, 0, ctx->stream>>>(ca);
    SBD_LAUNCHED(ctx, "cross_kernel_flat");
    return SBD_OK;
}

// Dense string sets: the same-spin streams carry only the singles' spectator-dependent term and
// the rest is added by two DGEMMs after the alpha side (sbd_samespin_gemm.cu).  Prepared lazily.
int dense_mode(sbd_ctx *ctx, bool *on) {
    *on = sbd_samespin_gemm_on(ctx);
    return *on ? sbd_samespin_gemm_prepare(ctx) : SBD_OK;
}

// Beta side for own alpha rows [r0, r1) (local): transpose those rows of x into
// X^T columns, then stream Y^T's column tiles covering them.  r0 is a
// multiple of kTW unless the whole range is launched.
int launch_beta_side(sbd_ctx *ctx, const double *x_own, i64 r0, i64 r1) {
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    const i64 rows = ctx->own_rows(), nb = B.n;
    if (r1 <= r0 || nb == 0) return SBD_OK;
    cudaStream_t st = ctx->stream;
    dim3 tg((unsigned)((nb + 31) / 32), (unsigned)((r1 - r0 + 31) / 32));
    transpose_kernel<<<tg, dim3(32, 8), 0, st>>>(x_own + r0 * nb, r1 - r0, nb, nb, ctx->xt.as<double>() + r0, ctx->ld_t);
    SBD_LAUNCHED(ctx, "transpose_kernel");
    SideArgs a{};
    a.n_rows = nb;
    a.row_base = 0;
    a.n_cols = rows;
    a.col_base = ctx->own_lo();
    a.X = ctx->xt.as<double>();
    a.ldx = ctx->ld_t;
    a.Y = ctx->yt.as<double>();
    a.ldy = ctx->ld_t;
    bool dense = false;
    if (int rc = dense_mode(ctx, &dense)) return rc;
    a.conn_off = dense ? B.s_off.as<int64_t>() : B.conn_off.as<int64_t>();
    a.conn = dense ? B.conn_j.as<Conn>() : B.conn.as<Conn>();
    a.J = A.J.as<double>();
    a.ldj = A.n;
    if (use_side_tma() && aligned16(a.X) && a.ldx % 2 == 0) {
        SBD_CUDA(ctx, sbd_smem_attr((const void *)side_kernel_async<false>, ctx->device, SideAsync<false>::smem()));
        a.tile0 = r0 / kTW;
        a.ytb = yt_blocked_enabled();
        ctx->yt_blocked = a.ytb;
        const i64 t1 = (r1 + kTW - 1) / kTW;
        dim3 g((unsigned)((nb + kRowsPerCta - 1) / kRowsPerCta), (unsigned)(t1 - a.tile0));
        side_kernel_async<false><<<g, kRowsPerCta * 32, SideAsync<false>::smem(), st>>>(a);
    } else {
        if (r0 != 0 || r1 != rows) return sbd_fail(ctx, SBD_EINVAL, "row-range beta side needs the aligned path");
        dim3 g((unsigned)((nb + kRowsPerCta - 1) / kRowsPerCta), (unsigned)((rows + kColsPerWarp - 1) / kColsPerWarp));
        ctx->yt_blocked = false;
        side_kernel<true, false><<<g, kRowsPerCta * 32, 0, st>>>(a);
    }
    SBD_LAUNCHED(ctx, "side_kernel<beta>");
    return SBD_OK;
}

// Alpha side (+ diagonal, task 0, beta side fold-in) for own rows [r0, r1) (local).
int launch_alpha_side(sbd_ctx *ctx, const double *x_full, double *y, i64 r0, i64 r1, bool with_t0 = true) {
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    const i64 nb = B.n, rows = r1 - r0;
    if (rows <= 0 || nb == 0) return SBD_OK;
    SideArgs a{};
    a.n_rows = rows;
    a.row_base = ctx->own_lo() + r0;
    a.n_cols = nb;
    a.col_base = 0;
    a.X = x_full;
    a.ldx = nb;
    a.Y = y + r0 * nb;
    a.ldy = nb;
    bool dense = false;
    if (int rc = dense_mode(ctx, &dense)) return rc;
    a.conn_off = dense ? A.s_off.as<int64_t>() : A.conn_off.as<int64_t>();
    a.conn = dense ? A.conn_j.as<Conn>() : A.conn.as<Conn>();
    a.J = B.J.as<double>();
    a.ldj = nb;
    a.ytb = ctx->yt_blocked;  // the layout the beta side wrote
    // the blocked Y^T groups alpha rows by 8: a chunk must start on a block (kTW-aligned chunks do)
    if (a.ytb && r0 % kRowsPerCta != 0) return sbd_fail(ctx, SBD_EINVAL, "alpha chunk start not a multiple of 8");
    a.YT = ctx->yt.as<double>() + (a.ytb ? r0 * nb : r0);
    a.ldyt = ctx->ld_t;
    a.diag = ctx->diag.as<double>() + r0 * nb;
    a.a_s_off = (with_t0 && A.ns > 0 && B.ns > 0) ? A.s_off.as<int64_t>() : nullptr;
    const bool vec = (nb % 2 == 0) && aligned16(x_full) && aligned16(y) && (r0 % 2 == 0);
    if (vec && use_side_tma()) {
        SBD_CUDA(ctx, sbd_smem_attr((const void *)side_kernel_async<true>, ctx->device, SideAsync<true>::smem()));
        dim3 gt((unsigned)((rows + kRowsPerCta - 1) / kRowsPerCta), (unsigned)((nb + kTW - 1) / kTW));
        side_kernel_async<true><<<gt, kRowsPerCta * 32, SideAsync<true>::smem(), ctx->stream>>>(a);
    } else {
        dim3 g((unsigned)((rows + kRowsPerCta - 1) / kRowsPerCta), (unsigned)((nb + kColsPerWarp - 1) / kColsPerWarp));
        if (vec) side_kernel<true, true><<<g, kRowsPerCta * 32, 0, ctx->stream>>>(a);
        else side_kernel<false, true><<<g, kRowsPerCta * 32, 0, ctx->stream>>>(a);
    }
    SBD_LAUNCHED(ctx, "side_kernel<alpha>");
    return SBD_OK;
}

// One pass of the partitioned alpha side (sbd_dist.cu): see SideArgs.seg_off.
int launch_alpha_pass(sbd_ctx *ctx, const double *X, double *y, const Conn *conn, const int64_t *seg_off, i64 stride,
                      int s_lo, int s_hi, i64 xo_row0, bool epi, bool acc_in) {
    const Sector &B = ctx->sec[1];
    const i64 nb = B.n, rows = ctx->own_rows();
    if (rows <= 0 || nb == 0) return SBD_OK;
    SideArgs a{};
    a.n_rows = rows;
    a.row_base = ctx->own_lo();
    a.n_cols = nb;
    a.col_base = 0;
    a.X = X;
    a.ldx = nb;
    a.Y = y;
    a.ldy = nb;
    a.conn = conn;
    a.J = B.J.as<double>();
    a.ldj = nb;
    a.ytb = ctx->yt_blocked;
    a.YT = ctx->yt.as<double>();
    a.ldyt = ctx->ld_t;
    a.diag = ctx->diag.as<double>();
    a.a_s_off = nullptr;  // task 0 is added after the last pass (sbd_cross_add)
    a.seg_off = seg_off;
    a.seg_stride = stride;
    a.seg_lo = s_lo;
    a.seg_hi = s_hi;
    a.xo_row0 = xo_row0;
    a.epi = epi;
    a.acc_in = acc_in;
    const bool vec = (nb % 2 == 0) && aligned16(X) && aligned16(y);
    if (vec && use_side_tma()) {
        SBD_CUDA(ctx, sbd_smem_attr((const void *)side_kernel_async<true, true>, ctx->device, SideAsync<true>::smem()));
        dim3 gt((unsigned)((rows + kRowsPerCta - 1) / kRowsPerCta), (unsigned)((nb + kTW - 1) / kTW));
        side_kernel_async<true, true><<<gt, kRowsPerCta * 32, SideAsync<true>::smem(), ctx->stream>>>(a);
    } else {
        dim3 g((unsigned)((rows + kRowsPerCta - 1) / kRowsPerCta), (unsigned)((nb + kColsPerWarp - 1) / kColsPerWarp));
        if (vec) side_kernel<true, true, true><<<g, kRowsPerCta * 32, 0, ctx->stream>>>(a);
        else side_kernel<false, true, true><<<g, kRowsPerCta * 32, 0, ctx->stream>>>(a);
    }
    SBD_LAUNCHED(ctx, "side_kernel<alpha pass>");
    return SBD_OK;
}

int ensure_events(sbd_ctx *ctx, size_t n) {
    if (!ctx->copy_stream) SBD_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    while (ctx->events.size() < n) {
        cudaEvent_t e;
        SBD_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->events.push_back(e);
    }
    return SBD_OK;
}

}  // namespace

// Dense string sets (sbd_samespin_gemm.cu): the auxiliary stream runs the two same-spin DGEMMs and
// then the beta stream (transpose + singles' J term) while the main stream runs task 0 (the longest
// kernel there); the alpha stream waits for both, and the DGEMMs' result is added last.
static int sigma_dense(sbd_ctx *ctx, const double *x_full, double *y) {
    int rc = require_product(ctx);
    if (rc) return rc;
    if ((rc = ensure_scratch(ctx)) || (rc = ensure_diag(ctx)) || (rc = sbd_samespin_gemm_prepare(ctx))) return rc;
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    if (ctx->own_rows() == 0 || B.n == 0) return SBD_OK;
    if ((rc = sbd_samespin_gemm_start(ctx, x_full))) return rc;
    cudaStream_t main = ctx->stream;
    ctx->stream = ctx->aux_stream;  // the beta stream after the DGEMMs, on the auxiliary stream
    rc = launch_beta_side(ctx, x_full + ctx->own_lo() * B.n, 0, ctx->own_rows());
    ctx->stream = main;
    if (rc) return rc;
    if ((rc = sbd_samespin_gemm_mark(ctx))) return rc;
    const bool additive = A.ns > 0 && B.ns > 0 && cross_additive(ctx);
    if (A.ns > 0 && B.ns > 0 && !additive && (rc = launch_cross(ctx, x_full, y))) return rc;
    SBD_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0));  // Y^T (and Z) ready
    if ((rc = launch_alpha_side(ctx, x_full, y, 0, ctx->own_rows(), !additive))) return rc;
    if (additive && (rc = launch_cross(ctx, x_full, y, true))) return rc;
    return sbd_samespin_gemm_finish(ctx, y);
}

int sbd_require_sigma_ready(sbd_ctx *ctx) {
    int rc = require_ready(ctx);
    if (rc) return rc;
    rc = require_product(ctx);
    if (rc) return rc;
    rc = ensure_scratch(ctx);
    if (rc) return rc;
    return ensure_diag(ctx);
}

int sbd_beta_side(sbd_ctx *ctx, const double *x_own) { return launch_beta_side(ctx, x_own, 0, ctx->own_rows()); }

int sbd_alpha_pass(sbd_ctx *ctx, const double *X, double *y, const Conn *conn, const int64_t *seg_off, i64 stride,
                   int s_lo, int s_hi, i64 xo_row0, bool epi, bool acc_in) {
    return launch_alpha_pass(ctx, X, y, conn, seg_off, stride, s_lo, s_hi, xo_row0, epi, acc_in);
}

int sbd_cross_add(sbd_ctx *ctx, const double *X, double *y, const SConn *sconn) {
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    if (ctx->own_rows() == 0 || B.n == 0 || A.ns == 0 || B.ns == 0) return SBD_OK;
    return launch_cross(ctx, X, y, true, sconn);
}

extern "C" {

int sbd_diag(sbd_ctx *ctx, double *out_dev) {
    SBD_CHECK_CTX(ctx);
    int rc = require_ready(ctx);
    if (rc) return rc;
    rc = ensure_diag(ctx);
    if (rc) return rc;
    const i64 n = ctx->explicit_mode ? ctx->n_det : ctx->own_rows() * ctx->sec[1].n;
    if (out_dev && n)
        SBD_CUDA(ctx, cudaMemcpyAsync(out_dev, ctx->diag.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    return SBD_OK;
}

int sbd_sigma_local(sbd_ctx *ctx, const double *x_own) {
    SBD_CHECK_CTX(ctx);
    int rc = require_ready(ctx);
    if (rc) return rc;
    rc = require_product(ctx);
    if (rc) return rc;
    rc = ensure_scratch(ctx);
    if (rc) return rc;
    return launch_beta_side(ctx, x_own, 0, ctx->own_rows());
}

int sbd_sigma_remote(sbd_ctx *ctx, const double *x_full, double *y) {
    SBD_CHECK_CTX(ctx);
    int rc = require_ready(ctx);
    if (rc) return rc;
    rc = require_product(ctx);
    if (rc) return rc;
    rc = ensure_diag(ctx);
    if (rc) return rc;
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    if (ctx->own_rows() == 0 || B.n == 0) return SBD_OK;
    const bool dense = sbd_samespin_gemm_on(ctx);
    if (dense) {  // the dense same-spin products run beside task 0 and the alpha stream
        if ((rc = sbd_samespin_gemm_prepare(ctx))) return rc;
        if ((rc = sbd_samespin_gemm_start(ctx, x_full))) return rc;
        if ((rc = sbd_samespin_gemm_mark(ctx))) return rc;
    }
    if (A.ns > 0 && B.ns > 0 && cross_additive(ctx)) {  // sparse singles: task 0 added afterwards
        rc = launch_alpha_side(ctx, x_full, y, 0, ctx->own_rows(), false);
        if (rc) return rc;
        rc = launch_cross(ctx, x_full, y, true);
    } else {
        if (A.ns > 0 && B.ns > 0) {  // task 0 exists only when both sectors have in-set singles
            rc = launch_cross(ctx, x_full, y);
            if (rc) return rc;
        }
        rc = launch_alpha_side(ctx, x_full, y, 0, ctx->own_rows());
    }
    if (rc) return rc;
    return dense ? sbd_samespin_gemm_finish(ctx, y) : SBD_OK;
}

int sbd_sigma(sbd_ctx *ctx, const double *x_full, double *y) {
    SBD_CHECK_CTX(ctx);
    SbdRange range("sbd/sigma");
    int rc = require_ready(ctx);
    if (rc) return rc;
    if (!x_full || !y) return sbd_fail(ctx, SBD_EINVAL, "null vector");
    if (ctx->explicit_mode) {
        rc = ensure_diag(ctx);
        if (rc) return rc;
        return sbd_explicit_sigma(ctx, x_full, y);
    }
    if (sbd_samespin_gemm_on(ctx)) return sigma_dense(ctx, x_full, y);
    rc = sbd_sigma_local(ctx, x_full + ctx->own_lo() * ctx->sec[1].n);
    if (rc) return rc;
    return sbd_sigma_remote(ctx, x_full, y);
}

int sbd_sigma_multi(sbd_ctx *ctx, const double *x_full, int64_t ldx, double *y, int64_t ldy, int nvec) {
    SBD_CHECK_CTX(ctx);
    if (nvec < 0) return sbd_fail(ctx, SBD_EINVAL, "nvec must be >= 0");
    const i64 nfull = ctx->explicit_mode ? ctx->n_det : ctx->sec[0].n * ctx->sec[1].n;
    const i64 nown = ctx->explicit_mode ? ctx->n_det : ctx->own_rows() * ctx->sec[1].n;
    if (nvec > 1 && (ldx < nfull || ldy < nown)) return sbd_fail(ctx, SBD_EINVAL, "leading dimension too small");
    for (int v = 0; v < nvec; ++v) {
        int rc = sbd_sigma(ctx, x_full + (i64)v * ldx, y + (i64)v * ldy);
        if (rc) return rc;
    }
    return SBD_OK;
}

// Host buffers in and out.  With one owner of all rows and the aligned
// kernels, the copies are pipelined with the kernels in kTW-aligned alpha-row
// chunks on a second stream: the beta side of chunk c (it only reads x rows
// of its own column tiles) runs while chunk c+1 is uploaded; after the last
// chunk, task 0 and the alpha side run chunk by chunk, each chunk's y going
// back to the host while the next chunk computes.  The host pointers should
// be pinned for the copies to be asynchronous.
int sbd_sigma_host(sbd_ctx *ctx, const double *x_host, double *y_host) {
    SBD_CHECK_CTX(ctx);
    SbdRange range("sbd/sigma_host");
    int rc = require_ready(ctx);
    if (rc) return rc;
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    const i64 nb = B.n;
    const i64 nfull = ctx->explicit_mode ? ctx->n_det : A.n * nb;
    const i64 rows = ctx->explicit_mode ? 0 : ctx->own_rows();
    const i64 nown = ctx->explicit_mode ? ctx->n_det : rows * nb;
    SBD_CUDA(ctx, ctx->hx.ensure(sizeof(double) * (nfull + 2)));
    SBD_CUDA(ctx, ctx->hy.ensure(sizeof(double) * (nown + 2)));
    double *dx = ctx->hx.as<double>(), *dy = ctx->hy.as<double>();
    const bool pipelined = !ctx->explicit_mode && rows == A.n && nb % 2 == 0 && use_side_tma() && rows > 2 * kTW &&
                           !(A.ns > 0 && B.ns > 0 && cross_additive(ctx)) && !sbd_samespin_gemm_on(ctx);
    if (!pipelined) {
        if (nfull) SBD_CUDA(ctx, cudaMemcpyAsync(dx, x_host, sizeof(double) * nfull, cudaMemcpyHostToDevice, ctx->stream));
        rc = sbd_sigma(ctx, dx, dy);
        if (rc) return rc;
        if (nown) SBD_CUDA(ctx, cudaMemcpyAsync(y_host, dy, sizeof(double) * nown, cudaMemcpyDeviceToHost, ctx->stream));
        SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        return SBD_OK;
    }
    rc = ensure_scratch(ctx);
    if (rc) return rc;
    rc = ensure_diag(ctx);
    if (rc) return rc;
    const i64 nch = sigma_host_chunks();
    const i64 step = std::max<i64>(kTW, (rows / nch + kTW - 1) / kTW * kTW);
    std::vector<i64> cut{0};
    while (cut.back() < rows) cut.push_back(std::min(rows, cut.back() + step));
    const size_t nc = cut.size() - 1;
    rc = ensure_events(ctx, 2 * nc + 1);
    if (rc) return rc;
    cudaStream_t cs = ctx->copy_stream;
    cudaEvent_t *ev = ctx->events.data();
    // the copy stream must not overwrite dx/dy while earlier work on the compute stream uses them
    SBD_CUDA(ctx, cudaEventRecord(ev[2 * nc], ctx->stream));
    SBD_CUDA(ctx, cudaStreamWaitEvent(cs, ev[2 * nc], 0));
    for (size_t c = 0; c < nc; ++c) {
        const i64 r0 = cut[c], r1 = cut[c + 1];
        SBD_CUDA(ctx, cudaMemcpyAsync(dx + r0 * nb, x_host + r0 * nb, sizeof(double) * (r1 - r0) * nb,
                                      cudaMemcpyHostToDevice, cs));
        SBD_CUDA(ctx, cudaEventRecord(ev[c], cs));
        SBD_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ev[c], 0));
        rc = launch_beta_side(ctx, dx, r0, r1);
        if (rc) return rc;
    }
    // task 0 chunk by chunk too: chunk 0's result (and its download) starts after its own rows'
    // task 0 instead of the whole matrix's (PCIe idles less between the upload and the download)
    for (size_t c = 0; c < nc; ++c) {
        const i64 r0 = cut[c], r1 = cut[c + 1];
        if (A.ns > 0 && B.ns > 0) {
            rc = launch_cross(ctx, dx, dy, false, nullptr, r0, r1);
            if (rc) return rc;
        }
        rc = launch_alpha_side(ctx, dx, dy, r0, r1);
        if (rc) return rc;
        SBD_CUDA(ctx, cudaEventRecord(ev[nc + c], ctx->stream));
        SBD_CUDA(ctx, cudaStreamWaitEvent(cs, ev[nc + c], 0));
        SBD_CUDA(ctx, cudaMemcpyAsync(y_host + r0 * nb, dy + r0 * nb, sizeof(double) * (r1 - r0) * nb,
                                      cudaMemcpyDeviceToHost, cs));
    }
    SBD_CUDA(ctx, cudaStreamSynchronize(cs));
    SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SBD_OK;
}

int sbd_last_task0(sbd_ctx *ctx, int *kind) {
    SBD_CHECK_CTX(ctx);
    if (!kind) return sbd_fail(ctx, SBD_EINVAL, "null output");
    *kind = ctx->last_task0;
    return SBD_OK;
}

int sbd_sigma_model(sbd_ctx *ctx, double *cbar, double *bytes) {
    SBD_CHECK_CTX(ctx);
    int rc = require_ready(ctx);
    if (rc) return rc;
    const Sector &A = ctx->sec[0];
    if (ctx->explicit_mode) {  // no streaming model: report in-set alpha moves per string
        if (cbar) *cbar = A.n ? (double)(A.ns + A.nd) / (double)A.n : 0.0;
        if (bytes) *bytes = 0.0;
        return SBD_OK;
    }
    double cb = A.n ? (double)(A.ns + A.nd) / (double)A.n : 0.0;
    if (cbar) *cbar = cb;
    if (bytes) *bytes = 8.0 * (double)ctx->own_rows() * (double)ctx->sec[1].n * (3.0 + cb);
    return SBD_OK;
}

}  // extern "C"
