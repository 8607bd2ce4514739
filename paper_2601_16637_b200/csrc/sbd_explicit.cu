// Explicit (full-bitstring) determinant bases.
//
// Reference: the explicit branch of HamiltonianApplier (apply.py:675-683,
// 696-703) and _explicit_row / _find_det (apply.py:323-426): for every
// determinant it enumerates all single/double moves of each spin and every
// alpha-single x beta-single pair, and probes each candidate by binary search
// over the (alpha, beta)-sorted determinant list.
//
// B200 formulation.  The determinant list is factored through its unique
// alpha and beta strings: sec[0]/sec[1] hold them, so the existing device
// excitation tables give the IN-SET moves of each string directly (no probe
// for candidates that are not selected strings), with the same per-entry
// coefficients (Conn records, J tables, pair-pair ERI) as the product path.
// A determinant is the pair (A, B) of string indices.  The list is radix-
// sorted by (A, B) once; group A's sorted B's are the only place a probe
// searches.  One warp per determinant: lanes take the alpha moves, the beta
// moves and the flattened alpha-single x beta-single pairs, each probe is a
// short binary search inside one group, and the row's sum is a fixed-order
// warp reduction (deterministic, no atomics).
#include <algorithm>

#include "sbd_internal.cuh"

namespace {

constexpr int kExplWarps = 8;

// key = A * n_b + B: lexicographic (A, B) order in the fewest radix passes
__global__ void det_keys_kernel(const int32_t *__restrict__ A, const int32_t *__restrict__ B, i64 n, i64 n_b,
                                u64 *__restrict__ keys) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = (u64)A[i] * (u64)n_b + (u64)B[i];
}

// groups of the (A, B)-sorted list; every alpha index owns at least one det
__global__ void det_groups_kernel(const u64 *__restrict__ sorted, i64 n, i64 n_alpha, i64 n_b,
                                  int32_t *__restrict__ grp_off, int32_t *__restrict__ grp_b, int *__restrict__ dup) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const u64 k = sorted[i];
    const int32_t a = (int32_t)(k / (u64)n_b);
    grp_b[i] = (int32_t)(k - (u64)a * (u64)n_b);
    if (i == 0 || (int32_t)(sorted[i - 1] / (u64)n_b) != a) grp_off[a] = (int32_t)i;
    if (i > 0 && sorted[i - 1] == k) *dup = 1;
    if (i == n - 1) grp_off[n_alpha] = (int32_t)n;
}

// caller index of det (a, b), or -1 (_find_det, apply.py:323-335, restricted to group a)
__device__ __forceinline__ int find_det(const int32_t *__restrict__ grp_off, const int32_t *__restrict__ grp_b,
                                        const int32_t *__restrict__ perm, int a, int b) {
    int lo = __ldg(grp_off + a), hi = __ldg(grp_off + a + 1);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(grp_b + mid) < b) lo = mid + 1;
        else hi = mid;
    }
    return (lo < __ldg(grp_off + a + 1) && __ldg(grp_b + lo) == b) ? __ldg(perm + lo) : -1;
}

struct ExplArgs {
    i64 n_det, n_a, n_b;
    const int32_t *A, *B;
    const int32_t *grp_off, *grp_b, *perm;
    const double *x, *diag;
    double *y;
    const int64_t *a_conn_off, *b_conn_off;
    const Conn *a_conn, *b_conn;
    const int64_t *a_s_off, *b_s_off;
    const SConn *a_sconn, *b_sconn;
    const double *Ja, *Jb;  // J[P][string] of the alpha / beta sector
    const double *vpp;      // sign-folded pair-pair ERI rows (sbd_context.cu)
    i64 ld;
};

__global__ void __launch_bounds__(kExplWarps * 32) explicit_sigma_kernel(ExplArgs a) {
    const int lane = threadIdx.x & 31;
    const i64 i = (i64)blockIdx.x * kExplWarps + (threadIdx.x >> 5);
    if (i >= a.n_det) return;
    const int A = a.A[i], B = a.B[i];
    double acc = 0.0;
    // alpha moves (beta fixed): coefficient c + phase * J_beta[P][B]
    for (i64 e = a.a_conn_off[A] + lane; e < a.a_conn_off[A + 1]; e += 32) {
        const Conn cn = a.a_conn[e];
        const int j = find_det(a.grp_off, a.grp_b, a.perm, cn.tgt, B);
        if (j >= 0) {
            double c = cn.c;
            if (cn.info != 0) c = fma(cn.info > 0 ? 1.0 : -1.0, __ldg(a.Jb + (i64)(abs(cn.info) - 1) * a.n_b + B), c);
            acc = fma(c, __ldg(a.x + j), acc);
        }
    }
    // beta moves (alpha fixed): coefficient c + phase * J_alpha[P][A]
    for (i64 e = a.b_conn_off[B] + lane; e < a.b_conn_off[B + 1]; e += 32) {
        const Conn cn = a.b_conn[e];
        const int j = find_det(a.grp_off, a.grp_b, a.perm, A, cn.tgt);
        if (j >= 0) {
            double c = cn.c;
            if (cn.info != 0) c = fma(cn.info > 0 ? 1.0 : -1.0, __ldg(a.Ja + (i64)(abs(cn.info) - 1) * a.n_a + A), c);
            acc = fma(c, __ldg(a.x + j), acc);
        }
    }
    // alpha-single x beta-single pairs: s_a s_b (Pa|Pb)
    const i64 sa0 = a.a_s_off[A], nsa = a.a_s_off[A + 1] - sa0;
    const i64 sb0 = a.b_s_off[B], nsb = a.b_s_off[B + 1] - sb0;
    for (i64 t = lane; t < nsa * nsb; t += 32) {
        const SConn ea = a.a_sconn[sa0 + t / nsb], eb = a.b_sconn[sb0 + t % nsb];
        const int j = find_det(a.grp_off, a.grp_b, a.perm, ea.tgt, eb.tgt);
        if (j >= 0) {
            const int Pa = abs(ea.info) - 1, Pb = abs(eb.info) - 1;
            const i64 row = (i64)(2 * Pa + (ea.info < 0)) * 2 * a.ld;  // (-1)^s_a (Pa|.) then its negation
            const double v = __ldg(a.vpp + row + Pb + (eb.info < 0 ? a.ld : 0));
            acc = fma(v, __ldg(a.x + j), acc);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) a.y[i] = fma(a.diag[i], a.x[i], acc);
}

// diagonal per det, the reference's operation order (apply.py:100-112)
__global__ void explicit_diag_kernel(i64 n, const int32_t *__restrict__ A, const int32_t *__restrict__ B,
                                     const u64 *__restrict__ astr, const u64 *__restrict__ bstr,
                                     const double *__restrict__ ea, const double *__restrict__ eb,
                                     const double *__restrict__ dpq, int norb, double e_core,
                                     double *__restrict__ out) {
    extern __shared__ double sd[];
    for (int t = threadIdx.x; t < norb * norb; t += blockDim.x) sd[t] = dpq[t];
    __syncthreads();
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const int a = A[i], b = B[i];
        const u64 aw = astr[a], bw = bstr[b];
        double e = __dadd_rn(__dadd_rn(e_core, ea[a]), eb[b]);
        for (u64 ta = aw; ta; ta &= ta - 1) {
            const int p = __ffsll((long long)ta) - 1;
            for (u64 tb = bw; tb; tb &= tb - 1) e = __dadd_rn(e, sd[p * norb + __ffsll((long long)tb) - 1]);
        }
        out[i] = e;
    }
}

}  // namespace

int sbd_build_explicit_index(sbd_ctx *ctx) {
    const i64 n = ctx->n_det;
    cudaStream_t st = ctx->stream;
    DevBuf keys, sorted, dup;
    SBD_CUDA(ctx, keys.ensure(sizeof(u64) * (n + 1)));
    SBD_CUDA(ctx, ctx->grp_off.ensure(sizeof(int32_t) * (ctx->sec[0].n + 1)));
    SBD_CUDA(ctx, ctx->grp_b.ensure(sizeof(int32_t) * (n + 1)));
    SBD_CUDA(ctx, dup.ensure(sizeof(int)));
    SBD_CUDA(ctx, cudaMemsetAsync(dup.p, 0, sizeof(int), st));
    const i64 na = ctx->sec[0].n, nb = std::max<i64>(1, ctx->sec[1].n);
    det_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(ctx->det_a.as<int32_t>(), ctx->det_b.as<int32_t>(), n, nb,
                                                      keys.as<u64>());
    SBD_LAUNCHED(ctx, "det keys");
    int kbits = 1;
    while (kbits < 64 && ((u64)1 << kbits) < (u64)na * (u64)nb) ++kbits;
    int rc = sbd_radix_sort(ctx, keys.as<u64>(), n, kbits, sorted, ctx->grp_perm);
    if (rc) return rc;
    det_groups_kernel<<<grid_for(n, 256), 256, 0, st>>>(sorted.as<u64>(), n, na, nb, ctx->grp_off.as<int32_t>(),
                                                        ctx->grp_b.as<int32_t>(), dup.as<int>());
    SBD_LAUNCHED(ctx, "det groups");
    int has_dup = 0;
    SBD_CUDA(ctx, cudaMemcpyAsync(&has_dup, dup.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    SBD_CUDA(ctx, cudaStreamSynchronize(st));
    if (has_dup) return sbd_fail(ctx, SBD_EINVAL, "duplicate determinants in explicit basis");
    ctx->explicit_built = true;
    return SBD_OK;
}

int sbd_explicit_diag(sbd_ctx *ctx, double *out) {
    const i64 n = ctx->n_det;
    if (n == 0) return SBD_OK;
    const size_t smem = sizeof(double) * ctx->norb * ctx->norb;
    const unsigned blocks = (unsigned)std::min<i64>(grid_for(n, 256), (i64)ctx->num_sms * 16);
    explicit_diag_kernel<<<blocks, 256, smem, ctx->stream>>>(
        n, ctx->det_a.as<int32_t>(), ctx->det_b.as<int32_t>(), ctx->sec[0].str.as<u64>(), ctx->sec[1].str.as<u64>(),
        ctx->sec[0].energy.as<double>(), ctx->sec[1].energy.as<double>(), ctx->dpq.as<double>(), ctx->norb,
        ctx->e_core, out);
    SBD_LAUNCHED(ctx, "explicit_diag_kernel");
    return SBD_OK;
}

int sbd_explicit_sigma(sbd_ctx *ctx, const double *x, double *y) {
    const Sector &SA = ctx->sec[0], &SB = ctx->sec[1];
    ExplArgs a{};
    a.n_det = ctx->n_det;
    a.n_a = SA.n;
    a.n_b = SB.n;
    a.A = ctx->det_a.as<int32_t>();
    a.B = ctx->det_b.as<int32_t>();
    a.grp_off = ctx->grp_off.as<int32_t>();
    a.grp_b = ctx->grp_b.as<int32_t>();
    a.perm = ctx->grp_perm.as<int32_t>();
    a.x = x;
    a.diag = ctx->diag.as<double>();
    a.y = y;
    a.a_conn_off = SA.conn_off.as<int64_t>();
    a.b_conn_off = SB.conn_off.as<int64_t>();
    a.a_conn = SA.conn.as<Conn>();
    a.b_conn = SB.conn.as<Conn>();
    a.a_s_off = SA.s_off.as<int64_t>();
    a.b_s_off = SB.s_off.as<int64_t>();
    a.a_sconn = SA.sconn.as<SConn>();
    a.b_sconn = SB.sconn.as<SConn>();
    a.Ja = SA.J.as<double>();
    a.Jb = SB.J.as<double>();
    a.vpp = ctx->vpp.as<double>();
    a.ld = ctx->ld_vpp;
    if (a.n_det == 0) return SBD_OK;
    explicit_sigma_kernel<<<grid_for(a.n_det, kExplWarps), kExplWarps * 32, 0, ctx->stream>>>(a);
    SBD_LAUNCHED(ctx, "explicit_sigma_kernel");
    return SBD_OK;
}

extern "C" {

int sbd_set_dets(sbd_ctx *ctx, const uint64_t *alpha, const uint64_t *beta, int64_t n, int n_alpha_elec,
                 int n_beta_elec) {
    SBD_CHECK_CTX(ctx);
    if (n < 0 || (n > 0 && (!alpha || !beta))) return sbd_fail(ctx, SBD_EINVAL, "bad determinant list");
    if (n >= (int64_t)INT32_MAX) return sbd_fail(ctx, SBD_EINVAL, "too many determinants");
    // unique strings per spin in first-seen order and dets as index pairs, on the device
    // (stable radix sort, run heads, runs re-sorted by first occurrence)
    if (!ctx->have_integrals) return sbd_fail(ctx, SBD_EINVAL, "set integrals before strings");
    SBD_CUDA(ctx, ctx->det_a.ensure(sizeof(int32_t) * (n + 1)));
    SBD_CUDA(ctx, ctx->det_b.ensure(sizeof(int32_t) * (n + 1)));
    std::vector<u64> uniq[2];
    for (int spin = 0; spin < 2; ++spin) {
        const uint64_t *src = spin ? beta : alpha;
        DevBuf keys, u;
        i64 nu = 0;
        SBD_CUDA(ctx, keys.ensure(sizeof(u64) * (n + 1)));
        if (n) SBD_CUDA(ctx, cudaMemcpy(keys.p, src, sizeof(u64) * n, cudaMemcpyHostToDevice));
        int rc = sbd_unique_first_seen_index(ctx, keys.as<u64>(), n, ctx->norb, u, &nu,
                                             spin ? ctx->det_b.as<int32_t>() : ctx->det_a.as<int32_t>());
        if (rc) return rc;
        uniq[spin].resize((size_t)nu);
        if (nu) SBD_CUDA(ctx, cudaMemcpy(uniq[spin].data(), u.p, sizeof(u64) * nu, cudaMemcpyDeviceToHost));
    }
    int rc = sbd_set_strings(ctx, 0, uniq[0].data(), (int64_t)uniq[0].size(), n_alpha_elec);
    if (rc) return rc;
    rc = sbd_set_strings(ctx, 1, uniq[1].data(), (int64_t)uniq[1].size(), n_beta_elec);
    if (rc) return rc;
    ctx->explicit_mode = true;
    ctx->explicit_built = false;
    ctx->n_det = n;
    ctx->diag_valid = false;
    return SBD_OK;
}

}  // extern "C"
