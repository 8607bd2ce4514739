// Internal declarations shared by the sbd_*.cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sbd.h"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for profilers (no-ops without one attached)

// Scoped NVTX range: sigma phases, table builds and Davidson iterations show up by name in
// Nsight Compute / Systems timelines (`ncu --nvtx --nvtx-include "sbd/"`).
struct SbdRange {
    explicit SbdRange(const char *name) { nvtxRangePushA(name); }
    ~SbdRange() { nvtxRangePop(); }
};

typedef uint64_t u64;
typedef int64_t i64;

// One kernel-ready connection of a source string (same-spin excitation).
//   info == 0      : double; coefficient c (spectator independent)
//   info == +-(P+1): single with orbital pair P = tri(p, r) and phase sign(info);
//                    c = phase * F, full coefficient c + phase * J[P][spectator]
struct __align__(16) Conn {
    int32_t tgt;
    int32_t info;
    double c;
};

// A bare single (for the opposite-spin alpha-single x beta-single term):
// info = phase * (P + 1).
struct __align__(8) SConn {
    int32_t tgt;
    int32_t info;
};

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    ~DevBuf() { release(); }
    void release();
    cudaError_t ensure(size_t nbytes);  // grow-only
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

struct Sector {
    i64 n = 0;
    int n_elec = 0;
    bool present = false;
    std::vector<u64> host;  // caller order
    DevBuf str;             // u64[n] caller order
    DevBuf sorted, perm;    // u64[n], int32[n]
    // reference-layout CSR (device)
    i64 ns = 0, nd = 0;
    DevBuf s_off, s_tgt, s_hole, s_part, s_phase;
    DevBuf d_off, d_tgt, d_h1, d_h2, d_p1, d_p2, d_phase;
    // kernel-ready
    DevBuf conn_off, conn;   // i64[n+1], Conn[ns+nd]
    DevBuf sconn;            // SConn[ns] (offsets = s_off)
    DevBuf s_row;            // int32[ns]: source string of each single
    DevBuf energy;           // f64[n]: same-spin diagonal energy per string
    DevBuf J;                // f64[npair][n]: J[P][i] = sum_{q in string i} (P|qq)
    // singles for the opposite-spin (task 0) kernel: chunked sliced ELL, see
    // build_sell (sbd_excite.cu) for the layout
    DevBuf sell_ent;         // u32[sell_nent]
    DevBuf sell_goff;        // int32[sell_h][groups+1]
    DevBuf sell_col;         // int32[groups*32]: string at each position (-1: padding)
    i64 sell_groups = 0, sell_nent = 0, sell_h = 1, sell_chunk = 0;
    std::vector<int32_t> sell_goff_host;  // host copy of sell_goff
    // dense-set mode (sbd_samespin_gemm.cu): spectator-independent coefficients as a dense n x n
    // matrix, and the singles (offsets s_off) with c = 0 for the spectator-dependent J term
    DevBuf dense, conn_j;
    int sell_pbits = 1;
    bool built = false;
};

// Alpha-block partition over ranks (sbd_dist.cu): NCCL communicator, the
// exchange plan and the pipelined pass schedule of sbd_sigma_dist.
//   x_work rows: segment 0 = the rank's own alpha rows, segment s (1..P-1) =
//   the rows needed from peer (rank - s) mod P, received at ring step s.  The
//   own rows' alpha connections are remapped to x_work rows and sorted by
//   that row, so the connections of one segment are one contiguous range
//   (seg_off[row * (P + 1) + s] .. [s + 1]) and a pass over the segments of
//   the steps that have landed is one contiguous range per row.
struct DistState {
    bool on = false;
    int rank = 0, nranks = 1;
    void *comm = nullptr;             // ncclComm_t
    cudaStream_t cs = nullptr;        // exchange stream
    std::vector<i64> blk;             // make_partition edges, P + 1
    bool planned = false;
    int sparse = 0;                   // 1: only referenced rows travel
    int group_steps = 2;              // ring steps per pipelined pass
    double needed_fraction = 1.0;     // max over ranks of (referenced remote rows / remote rows)
    std::vector<i64> seg_start;       // P + 1 (x_work row of each segment, last = work rows)
    std::vector<i64> recv_cnt;        // rows received at step s (s = 1..P-1), index s
    std::vector<i64> send_cnt, send_off;  // rows sent at step s to (rank + s) mod P, offsets in send_rows
    DevBuf xw;                        // x_work [work rows][n_beta]
    DevBuf conn;                      // own rows' Conn, remapped + sorted per row
    DevBuf seg_off;                   // i64[rows][P + 1]
    DevBuf sconn;                     // copy of alpha sconn, own entries remapped
    DevBuf send_rows, send_buf;       // sparse: local rows to pack per step, packed rows
    std::vector<cudaEvent_t> ev;      // sync events (one per group + start)
    // profiling (sbd_dist_set_profiling): timing events per group, accumulated per sigma
    bool profile = false;
    std::vector<cudaEvent_t> tev;
    bool tev_pending = false;
    i64 n_sigma = 0;
    std::vector<double> compute_ms, transfer_ms, exposed_ms;  // per step (0 = local, g = group g)
    double total_ms = 0.0;
};

// direct-CI task 0 (sbd_dci.cu): pair-pair ERI block and the beta singles re-sorted for the gather
struct DciState {
    bool valid = false;
    int nq = 0, nqp = 0, kp_max = 0, kb_max = 0, ld_e = 0, nt = 128, ntiles = 0, wmax = 0;
    DevBuf eq;    // f64 [npair][nqp]
    DevBuf ent;   // u32 [beta singles], per beta string sorted by target
    DevBuf toff;  // int32 [n_beta][ntiles + 1]
    DevBuf ell, woff, wt;  // per column tile: ELL block [wt][n_beta] of ent at woff (u32, i64, int32)
};

// device ingestion results (sbd_ingest.cu), first-seen order
struct IngestState {
    DevBuf det_a, det_b, det_count, alpha, beta;
    i64 n_det = 0, n_alpha = 0, n_beta = 0, n_samples = 0, n_kept = 0;
    bool ready = false;
};

struct sbd_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    int norb = 0;
    i64 npair = 0, n_eri = 0;
    double e_core = 0.0;
    bool have_integrals = false;
    DevBuf h, eri, dpq;  // h[norb*norb], eri, dpq[norb*norb] = (pp|qq)
    DevBuf vpp;          // sign-folded pair-pair ERI rows: row (P, sa) at (2P + sa) * 2 ld_vpp holds
                         //   [ (-1)^sa (P|Q) for Q < ld_vpp | -(-1)^sa (P|Q) for Q < ld_vpp ]
    i64 ld_vpp = 0;
    Sector sec[2];
    i64 row_lo = 0, row_hi = -1;  // owned alpha rows (row_hi < 0: all)
    // scratch for sigma
    DevBuf xt, yt;               // [n_beta][ld_t]; yt blocked by 8 alpha rows when yt_blocked (sbd_sigma.cu)
    i64 ld_t = 0;
    bool yt_blocked = false;
    DevBuf diag;                 // owned rows, cached
    bool diag_valid = false;
    DevBuf red;                  // reduction scratch
    DevBuf hx, hy;               // device staging for sbd_sigma_host
    cudaStream_t copy_stream = nullptr;  // sbd_sigma_host: H2D/D2H overlapped with the kernels
    std::vector<cudaEvent_t> events;
    int num_sms = 148;
    // explicit (full-bitstring) basis: dets are (A, B) pairs of unique-string
    // indices; sec[0]/sec[1] hold the unique alpha/beta strings (first-seen order)
    bool explicit_mode = false;
    i64 n_det = 0;
    DevBuf det_a, det_b;         // int32[n_det], caller order
    DevBuf grp_off;              // int32[n_alpha + 1]: dets sorted by (A, B), group of alpha A
    DevBuf grp_b, grp_perm;      // int32[n_det]: sorted B and caller index
    bool explicit_built = false;
    IngestState ingest;
    DistState dist;
    DciState dci;
    int last_task0 = 0;          // sbd_last_task0
    bool ssg_valid = false;      // same-spin dense matrices built (sbd_samespin_gemm.cu)
    void *cublas = nullptr;      // cublasHandle_t, created on first dense-set sigma
    cudaStream_t aux_stream = nullptr;    // dense-set DGEMMs, concurrent with the streams
    cudaEvent_t aux_ev[2] = {nullptr, nullptr};
    DevBuf ssg_z;                         // their result, added after the alpha side
    // 128-bit string list (norb <= 128): configuration processing + excitation tables only
    // (sbd_table128_*; U128 words in str/sorted)
    Sector t128;
    int t128_norb = 0;

    i64 own_lo() const { return row_lo; }
    i64 own_hi() const { return row_hi < 0 ? sec[0].n : row_hi; }
    i64 own_rows() const { return own_hi() - own_lo(); }
};

// Dynamic shared memory above 48 KB must be opted into per kernel and per device
// (a function attribute of the device's context): remember what each (kernel,
// device) pair was given, so a second GPU in the same process is set up too.
inline cudaError_t sbd_smem_attr(const void *func, int device, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, size_t> done;
    std::lock_guard<std::mutex> lock(mu);
    auto it = done.find({func, device});
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done[{func, device}] = bytes;
    return e;
}

// error helpers (sbd_context.cu)
int sbd_fail(sbd_ctx *ctx, int code, const std::string &msg);
int sbd_cuda_fail(sbd_ctx *ctx, cudaError_t e, const char *where);

#define SBD_CHECK_CTX(ctx)                                                   \
    do {                                                                     \
        if (!(ctx)) return sbd_fail(nullptr, SBD_EINVAL, "null context");    \
        cudaError_t _e = cudaSetDevice((ctx)->device);                       \
        if (_e != cudaSuccess) return sbd_cuda_fail((ctx), _e, "cudaSetDevice"); \
    } while (0)

#define SBD_CUDA(ctx, call)                                                  \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) return sbd_cuda_fail((ctx), _e, #call);       \
    } while (0)

#define SBD_LAUNCHED(ctx, name)                                              \
    do {                                                                     \
        cudaError_t _e = cudaGetLastError();                                 \
        if (_e != cudaSuccess) return sbd_cuda_fail((ctx), _e, name);        \
    } while (0)

// cross-TU entry points
int sbd_sort_strings(sbd_ctx *ctx, Sector &s);              // sbd_strings.cu
int sbd_build_sector_tables(sbd_ctx *ctx, Sector &s);       // sbd_excite.cu
int sbd_sort_strings128(sbd_ctx *ctx, Sector &s, int norb);             // sbd_strings.cu
int sbd_build_sector_tables128(sbd_ctx *ctx, Sector &s, int norb);      // sbd_excite.cu
int sbd_build_coefficients(sbd_ctx *ctx, Sector &s, const Sector &other);  // sbd_excite.cu
// LSD radix sort of n u64 keys (low key_bits significant) with the sort permutation (sbd_strings.cu)
int sbd_radix_sort(sbd_ctx *ctx, const u64 *keys, i64 n, int key_bits, DevBuf &sorted, DevBuf &perm);
int sbd_build_explicit_index(sbd_ctx *ctx);                 // sbd_explicit.cu
// unique keys in first-seen order + per-element position in that list (sbd_ingest.cu)
int sbd_unique_first_seen_index(sbd_ctx *ctx, const u64 *keys, i64 n, int key_bits, DevBuf &uniq, i64 *nuniq,
                                int32_t *index);
int sbd_explicit_diag(sbd_ctx *ctx, double *out);           // sbd_explicit.cu
int sbd_explicit_sigma(sbd_ctx *ctx, const double *x, double *y);  // sbd_explicit.cu
// sigma building blocks used by the partitioned sigma (sbd_sigma.cu)
int sbd_require_sigma_ready(sbd_ctx *ctx);                  // tables built, scratch + diag ready
int sbd_beta_side(sbd_ctx *ctx, const double *x_own);      // transpose + beta stream of the owned rows
// alpha stream over the connections seg_off[row*stride + s_lo] .. [row*stride + s_hi] of each owned row;
// epi: + diag o x + (B X^T)^T, y written; acc_in: y += (no epilogue)
int sbd_alpha_pass(sbd_ctx *ctx, const double *X, double *y, const Conn *conn, const int64_t *seg_off, i64 stride,
                   int s_lo, int s_hi, i64 xo_row0, bool epi, bool acc_in);
int sbd_cross_add(sbd_ctx *ctx, const double *X, double *y, const SConn *sconn);  // y += task 0
// same-spin parts as cuBLAS DGEMMs for dense string sets (sbd_samespin_gemm.cu)
bool sbd_samespin_gemm_on(const sbd_ctx *ctx);
int sbd_samespin_gemm_prepare(sbd_ctx *ctx);
int sbd_samespin_gemm_start(sbd_ctx *ctx, const double *x_full);
int sbd_samespin_gemm_mark(sbd_ctx *ctx);
int sbd_samespin_gemm_finish(sbd_ctx *ctx, double *y);
void sbd_samespin_gemm_release(sbd_ctx *ctx);
// direct-CI task 0 on the fp64 tensor cores (sbd_dci.cu): dense string sets
bool sbd_dci_eligible(sbd_ctx *ctx, const double *x_full);
int sbd_cross_dci(sbd_ctx *ctx, const double *x_full, double *y, bool additive, const SConn *sconn);
void sbd_dist_release(sbd_ctx *ctx);                        // sbd_dist.cu (called by sbd_destroy)
int sbd_dist_allreduce_internal(sbd_ctx *ctx, double *buf, i64 n, int op);  // 0 sum, 1 max, 2 min; no-op on 1 rank
int sbd_dist_check_internal(sbd_ctx *ctx);                  // NCCL asynchronous error -> SBD_ECUDA

// x rows of up to kSellWhole strings are staged whole (H = 1, cluster kernel);
// longer rows in chunks of at most kSellChunk strings (28 KB)
constexpr i64 kSellWhole = 12288;
constexpr i64 kSellChunk = 3584;
constexpr int kPackPairBits = 12;   // orbital pair index < 4096 (norb <= 64 gives 2080)
constexpr i64 kPackMaxStrings = (i64)1 << 19;  // target index in the remaining 19 bits

__host__ __device__ inline i64 tri_idx(i64 a, i64 b) {
    return a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a;
}

inline unsigned grid_for(i64 n, int block) {
    i64 g = (n + block - 1) / block;
    return (unsigned)(g < 1 ? 1 : g);
}
