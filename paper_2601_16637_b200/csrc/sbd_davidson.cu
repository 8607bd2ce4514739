// Device-resident Davidson building blocks (reference: davidson.py).
//
// The reference driver keeps V, W as lists of N-vectors and makes many
// separate passes per iteration (V.w, Ritz vectors, residuals, a full Gram
// matrix, two sequential MGS sweeps).  Here every pass over the subspace is a
// single fused streaming kernel that reads each of the k basis vectors once
// per element and reduces its dot products deterministically (per-block
// partials, then an ordered sum) -- the subspace work is HBM-bound, so the
// number of passes over V/W is the cost that matters:
//
//   sbd_vdots            T[:, k-1] = V^T w                          (davidson.py:248-249)
//   sbd_residual_precond r = Y^T W - theta Y^T V, t = precond(r),   (davidson.py:252-258,
//                        |r|^2, |t|^2 and V^T t in the same pass      159-163, 278)
//   sbd_gs_update        t -= V c ; V^T t ; |t|^2  (one CGS pass;    (davidson.py:166-185)
//                        two calls = CGS2 reorthogonalisation)
//   sbd_rotate           thick restart V <- V Y_keep in place       (davidson.py:280-289)
//   sbd_jacobi           projected k x k eigensolve, one warp       (davidson.py:86-148)
#include <algorithm>

#include "sbd_internal.cuh"

namespace {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Reduce acc[0..K) over the block and store to partial[blockIdx.x * K + i].
template <int K>
__device__ __forceinline__ void block_partials(const double (&acc)[K], double *__restrict__ partial) {
    __shared__ double sm[kWarps][K];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        double v = warp_sum(acc[i]);
        if (lane == 0) sm[w][i] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
        double s = 0.0;
        for (int ww = 0; ww < kWarps; ++ww) s += sm[ww][i];
        partial[(i64)blockIdx.x * K + i] = s;
    }
}

// Ordered sum of per-block partials (deterministic).  Output slot i < k reads
// partial slot i; slot i >= k reads partial slot kfix + (i - k), so kernels
// can keep a compile-time accumulator layout for a runtime subspace size.
__global__ void finish_partials(const double *__restrict__ partial, int nblocks, int stride, int k, int kfix,
                                int cnt, double *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const int src = i < k ? i : kfix + (i - k);
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += partial[(i64)b * stride + src];
    out[i] = s;
}

template <int K>
__global__ void __launch_bounds__(kBlock) vdots_kernel(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                       const double *__restrict__ w, double *__restrict__ partial) {
    double acc[K];
#pragma unroll
    for (int i = 0; i < K; ++i) acc[i] = 0.0;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
        const double we = __ldcs(w + e);
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) acc[i] = fma(__ldcs(V + i * ldv + e), we, acc[i]);
    }
    block_partials<K>(acc, partial);
}

// out[i] = V_i . w, out[K + i] = V_i . u  (one pass over V, two right-hand sides)
template <int K>
__global__ void __launch_bounds__(kBlock) vdots2_kernel(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                        const double *__restrict__ w, const double *__restrict__ u,
                                                        double *__restrict__ partial) {
    double acc[2 * K];
#pragma unroll
    for (int i = 0; i < 2 * K; ++i) acc[i] = 0.0;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
        const double we = __ldcs(w + e), ue = __ldg(u + e);
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) {
                const double v = __ldcs(V + i * ldv + e);
                acc[i] = fma(v, we, acc[i]);
                acc[K + i] = fma(v, ue, acc[K + i]);
            }
    }
    block_partials<2 * K>(acc, partial);
}

// K >= k; m <= 8 roots; jp = root whose preconditioned residual is projected
template <int K, int M>
__global__ void __launch_bounds__(kBlock)
residual_kernel(const double *__restrict__ V, const double *__restrict__ W, int k, i64 ldv, i64 n,
                const double *__restrict__ Y, const double *__restrict__ theta, int m, int jp,
                const double *__restrict__ diag, double delta, double *__restrict__ T, i64 ldt,
                double *__restrict__ partial) {
    __shared__ double ys[64 * 8];
    __shared__ double th[8];
    for (int i = threadIdx.x; i < k * m; i += blockDim.x) ys[i] = Y[i];
    if (threadIdx.x < m) th[threadIdx.x] = theta[threadIdx.x];
    __syncthreads();
    // accumulator layout: [0,K) V^T t_jp | K: |t_jp|^2 | K+1+j: |r_j|^2
    double acc[K + 1 + M];
#pragma unroll
    for (int i = 0; i < K + 1 + M; ++i) acc[i] = 0.0;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
        double u[M], wy[M];
#pragma unroll
        for (int j = 0; j < M; ++j) u[j] = wy[j] = 0.0;
        // Ritz vector and image components (davidson.py:256-257): u = Y^T V, wy = Y^T W
#pragma unroll
        for (int i = 0; i < K; ++i) {
            if (i < k) {
                const double v = V[i * ldv + e], ww = __ldcs(W + i * ldv + e);
#pragma unroll
                for (int j = 0; j < M; ++j)
                    if (j < m) {
                        u[j] = fma(ys[i * m + j], v, u[j]);
                        wy[j] = fma(ys[i * m + j], ww, wy[j]);
                    }
            }
        }
        const double d = diag[e];
        double tj = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            if (j < m) {
                const double r = wy[j] - th[j] * u[j];
                acc[K + 1 + j] = fma(r, r, acc[K + 1 + j]);
                // precondition (davidson.py:159-163): sign(0) = +1, clamp at delta
                const double g = d - th[j];
                const double den = (g >= 0.0 ? 1.0 : -1.0) * fmax(fabs(g), delta);
                const double t = r / den;
                T[j * ldt + e] = t;
                if (j == jp) tj = t;
            }
        }
        acc[K] = fma(tj, tj, acc[K]);
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) acc[i] = fma(V[i * ldv + e], tj, acc[i]);
    }
    block_partials<K + 1 + M>(acc, partial);
}

// t -= sum_i c_i V_i ; then partial dots V_i . t (i < kdot) and |t|^2 (slot kdot)
template <int K>
__global__ void __launch_bounds__(kBlock) gs_kernel(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                    const double *__restrict__ c, int kdot, double *__restrict__ t,
                                                    double *__restrict__ partial) {
    __shared__ double cs[K];
    for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = c[i];
    __syncthreads();
    double acc[K + 1];
#pragma unroll
    for (int i = 0; i <= K; ++i) acc[i] = 0.0;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
        double te = t[e];
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) te = fma(-cs[i], V[i * ldv + e], te);
        t[e] = te;
        // second touch of the same V lines: served by L1
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < kdot) acc[i] = fma(__ldg(V + i * ldv + e), te, acc[i]);
        acc[K] = fma(te, te, acc[K]);
    }
    block_partials<K + 1>(acc, partial);
}

__global__ void scale_copy_kernel(const double *__restrict__ src, double *__restrict__ dst, i64 n,
                                  const double *__restrict__ s) {
    const double f = *s;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x)
        dst[e] = src[e] * f;
}

// in place: V[:, j] <- sum_i Y[i, j] V[:, i]  for j < keep (per element independent)
template <int K>
__global__ void __launch_bounds__(kBlock) rotate_kernel(double *__restrict__ V, int k, i64 ldv, i64 n,
                                                        const double *__restrict__ Y, int keep) {
    __shared__ double ys[K * K];
    for (int i = threadIdx.x; i < k * keep; i += blockDim.x) ys[i] = Y[i];
    __syncthreads();
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
        double v[K];
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) v[i] = V[i * ldv + e];
        for (int j = 0; j < keep; ++j) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < K; ++i)
                if (i < k) s = fma(ys[i * keep + j], v[i], s);
            V[j * ldv + e] = s;
        }
    }
}

template <int K>
__global__ void __launch_bounds__(kBlock) combine_kernel(const double *__restrict__ V, int k, i64 ldv, i64 n,
                                                         const double *__restrict__ Y, int m, double *__restrict__ U,
                                                         i64 ldu) {
    __shared__ double ys[K * 8];
    for (int i = threadIdx.x; i < k * m; i += blockDim.x) ys[i] = Y[i];
    __syncthreads();
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (i64)gridDim.x * blockDim.x) {
        double u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = 0.0;
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (i < k) {
                const double v = V[i * ldv + e];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < m) u[j] = fma(ys[i * m + j], v, u[j]);
            }
        for (int j = 0; j < m; ++j) U[j * ldu + e] = u[j];
    }
}

// Cyclic Jacobi (davidson.py:86-148) by one warp; lanes own matrix rows.
constexpr int kJacMax = 64;
__global__ void jacobi_kernel(const double *__restrict__ Ain, int k, int lda, double *__restrict__ evals,
                              double *__restrict__ evecs, int max_sweeps, int *__restrict__ info) {
    extern __shared__ double jsm[];
    double(*a)[kJacMax + 1] = reinterpret_cast<double(*)[kJacMax + 1]>(jsm);
    double(*v)[kJacMax + 1] = reinterpret_cast<double(*)[kJacMax + 1]>(jsm + kJacMax * (kJacMax + 1));
    int *order = reinterpret_cast<int *>(jsm + 2 * kJacMax * (kJacMax + 1));
    const int lane = threadIdx.x;
    // symmetrise: a = (M + M^T) / 2 ; v = I
    for (int idx = lane; idx < k * k; idx += 32) {
        int p = idx / k, q = idx % k;
        a[p][q] = (Ain[p * lda + q] + Ain[q * lda + p]) / 2.0;
        v[p][q] = p == q ? 1.0 : 0.0;
    }
    __syncwarp();
    double fro = 0.0;
    for (int idx = lane; idx < k * k; idx += 32) fro = fma(a[idx / k][idx % k], a[idx / k][idx % k], fro);
    fro = warp_sum(fro);
    const double tol = 1e-14 * sqrt(fro);
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        double off = 0.0;
        for (int p = lane; p < k - 1; p += 32)
            for (int q = p + 1; q < k; ++q) off += 2.0 * a[p][q] * a[p][q];
        off = warp_sum(off);
        if (sqrt(off) <= tol) break;
        for (int p = 0; p < k - 1; ++p) {
            for (int q = p + 1; q < k; ++q) {
                const double apq = a[p][q];
                if (apq == 0.0) continue;
                const double app = a[p][p], aqq = a[q][q];
                const double theta = (aqq - app) / (2.0 * apq);
                double t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
                if (theta < 0.0) t = -t;
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                __syncwarp();
                for (int r = lane; r < k; r += 32) {
                    if (r != p && r != q) {
                        const double arp = a[r][p], arq = a[r][q];
                        const double np = c * arp - s * arq, nq = s * arp + c * arq;
                        a[r][p] = np;
                        a[p][r] = np;
                        a[r][q] = nq;
                        a[q][r] = nq;
                    }
                    const double vrp = v[r][p], vrq = v[r][q];
                    v[r][p] = c * vrp - s * vrq;
                    v[r][q] = s * vrp + c * vrq;
                }
                if (lane == 0) {
                    a[p][p] = app - t * apq;
                    a[q][q] = aqq + t * apq;
                    a[p][q] = 0.0;
                    a[q][p] = 0.0;
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    if (lane == 0) {
        // stable ascending order of the diagonal (np.argsort kind="stable")
        for (int i = 0; i < k; ++i) order[i] = i;
        for (int i = 1; i < k; ++i) {
            int oi = order[i];
            double key = a[oi][oi];
            int j = i - 1;
            while (j >= 0 && a[order[j]][order[j]] > key) {
                order[j + 1] = order[j];
                --j;
            }
            order[j + 1] = oi;
        }
        info[0] = sweep;
    }
    __syncwarp();
    for (int i = lane; i < k; i += 32) evals[i] = a[order[i]][order[i]];
    for (int idx = lane; idx < k * k; idx += 32) {
        int r = idx / k, cidx = idx % k;
        evecs[r * k + cidx] = v[r][order[cidx]];
    }
}

int red_blocks(sbd_ctx *ctx, i64 n) {
    i64 b = (n + kBlock - 1) / kBlock;
    return (int)std::max<i64>(1, std::min<i64>(b, (i64)ctx->num_sms * 4));
}

int ensure_red(sbd_ctx *ctx, int nblocks, int stride) {
    SBD_CUDA(ctx, ctx->red.ensure(sizeof(double) * (size_t)nblocks * stride + 64));
    return SBD_OK;
}

int check_k(sbd_ctx *ctx, int k) {
    if (k < 0 || k > 64) return sbd_fail(ctx, SBD_EINVAL, "subspace size must be in [0, 64]");
    return SBD_OK;
}

template <template <int> class Launch, class... Args>
int dispatch_k(int k, Args... args) {
    if (k <= 8) return Launch<8>::run(args...);
    if (k <= 16) return Launch<16>::run(args...);
    if (k <= 32) return Launch<32>::run(args...);
    return Launch<64>::run(args...);
}

template <int K>
struct VdotsL {
    static int run(sbd_ctx *ctx, const double *V, int k, i64 ldv, i64 n, const double *w, double *out) {
        int nb = red_blocks(ctx, n);
        if (int rc = ensure_red(ctx, nb, K)) return rc;
        vdots_kernel<K><<<nb, kBlock, 0, ctx->stream>>>(V, k, ldv, n, w, ctx->red.as<double>());
        finish_partials<<<1, 64, 0, ctx->stream>>>(ctx->red.as<double>(), nb, K, k, K, k, out);
        SBD_LAUNCHED(ctx, "vdots");
        return SBD_OK;
    }
};

template <int K>
struct Vdots2L {
    static int run(sbd_ctx *ctx, const double *V, int k, i64 ldv, i64 n, const double *w, const double *u,
                   double *out) {
        int nb = red_blocks(ctx, n);
        if (int rc = ensure_red(ctx, nb, 2 * K)) return rc;
        vdots2_kernel<K><<<nb, kBlock, 0, ctx->stream>>>(V, k, ldv, n, w, u, ctx->red.as<double>());
        finish_partials<<<1, 64, 0, ctx->stream>>>(ctx->red.as<double>(), nb, 2 * K, k, K, k, out);
        finish_partials<<<1, 64, 0, ctx->stream>>>(ctx->red.as<double>() + K, nb, 2 * K, k, K, k, out + k);
        SBD_LAUNCHED(ctx, "vdots2");
        return SBD_OK;
    }
};

template <int K>
struct ResidL {
    template <int M>
    static void launch(sbd_ctx *ctx, int nb, const double *V, const double *W, int k, i64 ldv, i64 n,
                       const double *Y, const double *theta, int m, int jp, const double *diag, double delta,
                       double *T, i64 ldt) {
        residual_kernel<K, M><<<nb, kBlock, 0, ctx->stream>>>(V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T, ldt,
                                                             ctx->red.as<double>());
    }
    static int run(sbd_ctx *ctx, const double *V, const double *W, int k, i64 ldv, i64 n, const double *Y,
                   const double *theta, int m, int jp, const double *diag, double delta, double *T, i64 ldt,
                   double *out) {
        int nb = red_blocks(ctx, n);
        if (int rc = ensure_red(ctx, nb, K + 9)) return rc;
        if (m == 1) launch<1>(ctx, nb, V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T, ldt);
        else if (m == 2) launch<2>(ctx, nb, V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T, ldt);
        else if (m <= 4) launch<4>(ctx, nb, V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T, ldt);
        else launch<8>(ctx, nb, V, W, k, ldv, n, Y, theta, m, jp, diag, delta, T, ldt);
        const int stride = K + 1 + (m == 1 ? 1 : m == 2 ? 2 : m <= 4 ? 4 : 8);
        finish_partials<<<1, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nb, stride, k, K, k + 1 + m, out);
        SBD_LAUNCHED(ctx, "residual_precond");
        return SBD_OK;
    }
};

template <int K>
struct GsL {
    static int run(sbd_ctx *ctx, const double *V, int k, i64 ldv, i64 n, const double *c, int kdot, double *t,
                   double *out) {
        int nb = red_blocks(ctx, n);
        if (int rc = ensure_red(ctx, nb, K + 1)) return rc;
        gs_kernel<K><<<nb, kBlock, 0, ctx->stream>>>(V, k, ldv, n, c, kdot, t, ctx->red.as<double>());
        finish_partials<<<1, 128, 0, ctx->stream>>>(ctx->red.as<double>(), nb, K + 1, kdot, K, kdot + 1, out);
        SBD_LAUNCHED(ctx, "gs_update");
        return SBD_OK;
    }
};

template <int K>
struct RotL {
    static int run(sbd_ctx *ctx, double *V, int k, i64 ldv, i64 n, const double *Y, int keep) {
        rotate_kernel<K><<<red_blocks(ctx, n) * 2, kBlock, 0, ctx->stream>>>(V, k, ldv, n, Y, keep);
        SBD_LAUNCHED(ctx, "rotate");
        return SBD_OK;
    }
};

template <int K>
struct CombL {
    static int run(sbd_ctx *ctx, const double *V, int k, i64 ldv, i64 n, const double *Y, int m, double *U, i64 ldu) {
        combine_kernel<K><<<red_blocks(ctx, n) * 2, kBlock, 0, ctx->stream>>>(V, k, ldv, n, Y, m, U, ldu);
        SBD_LAUNCHED(ctx, "combine");
        return SBD_OK;
    }
};

}  // namespace

extern "C" {

int sbd_vdots(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *w, double *out) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (k == 0) return SBD_OK;
    return dispatch_k<VdotsL>(k, ctx, V, k, (i64)ldv, (i64)n, w, out);
}

int sbd_vdots2(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *w, const double *u,
               double *out) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (k == 0) return SBD_OK;
    if (k > 32) {  // keep accumulators in registers: two single-RHS passes
        if (int rc = dispatch_k<VdotsL>(k, ctx, V, k, (i64)ldv, (i64)n, w, out)) return rc;
        return dispatch_k<VdotsL>(k, ctx, V, k, (i64)ldv, (i64)n, u, out + k);
    }
    return dispatch_k<Vdots2L>(k, ctx, V, k, (i64)ldv, (i64)n, w, u, out);
}

int sbd_residual_precond(sbd_ctx *ctx, const double *V, const double *W, int k, int64_t ldv, int64_t n,
                         const double *Y, const double *theta, int m, const double *diag, double delta, double *T,
                         int64_t ldt, double *rn2, double *proj) {
    // rn2/proj: single output buffer of k + 1 + m doubles laid out as
    // [V^T t_0 (k) | |t_0|^2 | |r_j|^2 (m)]; `rn2` must equal proj + k + 1.
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (m < 1 || m > 8 || m > k) return sbd_fail(ctx, SBD_EINVAL, "n_roots must be in [1, min(8, k)]");
    if (rn2 != proj + k + 1) return sbd_fail(ctx, SBD_EINVAL, "rn2 must alias proj + k + 1");
    return dispatch_k<ResidL>(k, ctx, V, W, k, (i64)ldv, (i64)n, Y, theta, m, 0, diag, delta, T, (i64)ldt, proj);
}

int sbd_residual_precond_target(sbd_ctx *ctx, const double *V, const double *W, int k, int64_t ldv, int64_t n,
                                const double *Y, const double *theta, int m, int target, const double *diag,
                                double delta, double *T, int64_t ldt, double *out) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (m < 1 || m > 8 || m > k) return sbd_fail(ctx, SBD_EINVAL, "n_roots must be in [1, min(8, k)]");
    if (target < 0 || target >= m) return sbd_fail(ctx, SBD_EINVAL, "bad target root");
    return dispatch_k<ResidL>(k, ctx, V, W, k, (i64)ldv, (i64)n, Y, theta, m, target, diag, delta, T, (i64)ldt, out);
}

int sbd_gs_update(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *c, double *t,
                  double *out2) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (k == 0) {
        // only |t|^2
        return GsL<8>::run(ctx, V, 0, (i64)ldv, (i64)n, c, 0, t, out2);
    }
    return dispatch_k<GsL>(k, ctx, V, k, (i64)ldv, (i64)n, c, k, t, out2);
}

int sbd_gs_update_nodots(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *c, double *t,
                         double *out_norm2) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (k == 0) return GsL<8>::run(ctx, V, 0, (i64)ldv, (i64)n, c, 0, t, out_norm2);
    return dispatch_k<GsL>(k, ctx, V, k, (i64)ldv, (i64)n, c, 0, t, out_norm2);
}

int sbd_scale_copy(sbd_ctx *ctx, const double *src, double *dst, int64_t n, const double *scale) {
    SBD_CHECK_CTX(ctx);
    scale_copy_kernel<<<red_blocks(ctx, n) * 2, kBlock, 0, ctx->stream>>>(src, dst, n, scale);
    SBD_LAUNCHED(ctx, "scale_copy");
    return SBD_OK;
}

int sbd_rotate(sbd_ctx *ctx, double *V, int k, int64_t ldv, int64_t n, const double *Y, int keep) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (keep < 1 || keep > k) return sbd_fail(ctx, SBD_EINVAL, "keep must be in [1, k]");
    return dispatch_k<RotL>(k, ctx, V, k, (i64)ldv, (i64)n, Y, keep);
}

int sbd_combine(sbd_ctx *ctx, const double *V, int k, int64_t ldv, int64_t n, const double *Y, int m, double *U,
                int64_t ldu) {
    SBD_CHECK_CTX(ctx);
    if (int rc = check_k(ctx, k)) return rc;
    if (m < 1 || m > 8) return sbd_fail(ctx, SBD_EINVAL, "m must be in [1, 8]");
    return dispatch_k<CombL>(k, ctx, V, k, (i64)ldv, (i64)n, Y, m, U, (i64)ldu);
}

int sbd_jacobi(sbd_ctx *ctx, const double *A, int k, int lda, double *evals, double *evecs, int max_sweeps,
               int *info) {
    SBD_CHECK_CTX(ctx);
    if (k < 1 || k > kJacMax) return sbd_fail(ctx, SBD_EINVAL, "jacobi size must be in [1, 64]");
    const int smem = (int)(sizeof(double) * 2 * kJacMax * (kJacMax + 1) + sizeof(int) * kJacMax);
    static bool attr_set = false;
    if (!attr_set) {
        SBD_CUDA(ctx, cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_set = true;
    }
    jacobi_kernel<<<1, 32, smem, ctx->stream>>>(A, k, lda, evals, evecs, max_sweeps, info);
    SBD_LAUNCHED(ctx, "jacobi");
    return SBD_OK;
}

}  // extern "C"
