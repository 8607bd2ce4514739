// Native Davidson driver: sbd_davidson (reference davidson_solve, davidson.py:191-306).
//
// The same algorithm as the Python driver (paper_2601_16637_b200/davidson.py,
// which mirrors the reference step for step), with the host control loop in
// C++ so a C caller can solve without Python and the per-iteration host work
// is a few microseconds.  Every pass over the subspace is one of the fused
// kernels in sbd_davidson.cu; the sigma is the context's own operator
// (sbd_sigma: product or explicit basis, all rows owned).  Per iteration the
// host reads back one packed vector (Ritz values, residual norms, |t|^2,
// Jacobi sweeps, orthogonality loss and the speculative CGS pass-1 dots).
//
// The only departure from the Python driver: breakdown recovery draws its
// random direction on the device (counter-based hash + Box-Muller) instead of
// numpy's default_rng stream (davidson.py:295).  Breakdowns only occur when
// the correction lies in span(V); the recovered direction is orthogonalised
// against V either way.

#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "sbd_internal.cuh"

namespace {

constexpr int kMaxK = 64;
constexpr int kMaxRoots = 8;
constexpr int kMaxSweeps = 64;

// T[:, k-1] = T[k-1, :] = small[0:k]; G likewise from small[k:2k]
__global__ void set_tg_kernel(double *T, double *G, const double *small, int k, int ld) {
    int i = threadIdx.x;
    if (i < k) {
        T[i * ld + k - 1] = small[i];
        T[(k - 1) * ld + i] = small[i];
        G[i * ld + k - 1] = small[k + i];
        G[(k - 1) * ld + i] = small[k + i];
    }
}

// Y[i, j] = evecs[i, j] (k x k row-major) for j < mk; theta[j] = evals[j]
__global__ void ritz_prep_kernel(const double *evecs, const double *evals, int k, int mk, double *Y, double *theta) {
    for (int e = threadIdx.x; e < k * mk; e += blockDim.x) {
        int i = e / mk, j = e - i * mk;
        Y[e] = evecs[i * k + j];
    }
    if ((int)threadIdx.x < mk) theta[threadIdx.x] = evals[threadIdx.x];
}

// packed read-back: theta | residual^2 | |t|^2 | sweeps | ortho | [V^T t' | |t'|^2]
__global__ void pack_kernel(const double *evals, const double *small, const double *small2, const int *info,
                            const double *G, int ldg, int k, int mk, int track, int spec, double *pack) {
    __shared__ double red[256];
    int tid = threadIdx.x;
    double s = 0.0;
    if (track) {
        for (int e = tid; e < k * k; e += blockDim.x) {
            int i = e / k, j = e - i * k;
            double d = G[i * ldg + j] - (i == j ? 1.0 : 0.0);
            s += d * d;
        }
    }
    red[tid] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (tid < w) red[tid] += red[tid + w];
        __syncthreads();
    }
    if (tid < mk) {
        pack[tid] = evals[tid];
        pack[mk + tid] = small[k + 1 + tid];
    }
    if (tid == 0) {
        pack[2 * mk] = small[k];
        pack[2 * mk + 1] = (double)info[0];
        pack[2 * mk + 2] = track ? sqrt(red[0]) : 0.0;
    }
    if (spec && tid <= k) pack[2 * mk + 3 + tid] = small2[tid];
}

__global__ void copy_small_kernel(const double *src, double *dst, int n) {
    if ((int)threadIdx.x < n) dst[threadIdx.x] = src[threadIdx.x];
}

__global__ void set_scalar_kernel(double *p, double v) { *p = v; }

// thick restart bookkeeping: T = diag(evals[:keep]), G[:keep,:keep] = Gnew, c[:keep] = cnew
__global__ void restart_kernel(double *T, double *G, int ld, const double *evals, const double *rs, int keep,
                               double *c) {
    for (int e = threadIdx.x; e < ld * ld; e += blockDim.x) {
        int i = e / ld, j = e - i * ld;
        T[e] = (i == j && i < keep) ? evals[i] : 0.0;
        G[e] = (i < keep && j < keep) ? rs[i * keep + j] : 0.0;
    }
    if ((int)threadIdx.x < keep) c[threadIdx.x] = rs[keep * keep + threadIdx.x];
}

// Y (k x keep) from the first keep eigenvector columns
__global__ void cols_kernel(const double *evecs, int k, int keep, double *Y) {
    for (int e = threadIdx.x; e < k * keep; e += blockDim.x) {
        int i = e / keep, j = e - i * keep;
        Y[e] = evecs[i * k + j];
    }
}

// argmin of d[0:n] (first index on ties), two levels; the second level also
// writes the unit start vector v = e_argmin (davidson.py:219-221)
constexpr int kArgBlock = 256;

__device__ inline void better(double &bv, i64 &bi, double v, i64 i) {
    if (v < bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
    }
}

__global__ void argmin_partial_kernel(const double *d, i64 n, double *pv, i64 *pi) {
    __shared__ double sv[kArgBlock];
    __shared__ i64 si[kArgBlock];
    double bv = INFINITY;
    i64 bi = n;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        better(bv, bi, d[i], i);
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) better(sv[threadIdx.x], si[threadIdx.x], sv[threadIdx.x + w], si[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pv[blockIdx.x] = sv[0];
        pi[blockIdx.x] = si[0];
    }
}

__global__ void argmin_final_kernel(const double *pv, const i64 *pi, int nb, i64 n, double *v0) {
    __shared__ double sv[kArgBlock];
    __shared__ i64 si[kArgBlock];
    double bv = INFINITY;
    i64 bi = n;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) better(bv, bi, pv[i], pi[i]);
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) better(sv[threadIdx.x], si[threadIdx.x], sv[threadIdx.x + w], si[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) v0[si[0] < n ? si[0] : 0] = 1.0;
}

// partitioned start vector: local best (value, global index) -> s[0], s[1]
__global__ void argmin_local_kernel(const double *pv, const i64 *pi, int nb, i64 n, i64 goff, double *s) {
    __shared__ double sv[kArgBlock];
    __shared__ i64 si[kArgBlock];
    double bv = INFINITY;
    i64 bi = n;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) better(bv, bi, pv[i], pi[i]);
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) better(sv[threadIdx.x], si[threadIdx.x], sv[threadIdx.x + w], si[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        s[0] = sv[0];
        s[1] = si[0] < n ? (double)(goff + si[0]) : INFINITY;
        s[2] = sv[0];  // all-reduced (min) next
    }
}
// after s[2] = global min value: candidate index s[3] (all-reduced min next)
__global__ void argmin_candidate_kernel(double *s) { s[3] = s[0] == s[2] ? s[1] : INFINITY; }
// s[3] = global argmin (first index on ties, davidson.py:219-221): set it if it is local
__global__ void argmin_set_kernel(const double *s, i64 n, i64 goff, double *v0) {
    const double gi = s[3];
    if (gi >= (double)goff && gi < (double)(goff + n)) v0[(i64)gi - goff] = 1.0;
    else if (!(gi < INFINITY) && goff == 0) v0[0] = 1.0;  // no finite diagonal anywhere: e_0
}

__device__ inline u64 splitmix64(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// element i of the local slice is global element goff + i: the draw does not depend on the partition
__global__ void random_normal_kernel(double *t, i64 n, i64 goff, u64 seed) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const u64 gi = (u64)(goff + i);
        u64 a = splitmix64(seed ^ (2 * gi)), b = splitmix64(seed ^ (2 * gi + 1));
        double u1 = ((a >> 11) + 1) * 0x1.0p-53;  // (0, 1]
        double u2 = (b >> 11) * 0x1.0p-53;
        t[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
}

// RAII pinned host block
struct Pinned {
    double *p = nullptr;
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

struct Solver {
    sbd_ctx *ctx;
    sbd_davidson_opts o;
    i64 n = 0, ld = 0;
    int m = 1, kmax = 1, keep = 1;
    DevBuf vw, aux, diag, part;
    double *V = nullptr, *W = nullptr, *Tv = nullptr;
    double *small = nullptr, *small2 = nullptr, *scale = nullptr, *T = nullptr, *G = nullptr, *Y = nullptr,
           *Yk = nullptr, *th = nullptr, *jw = nullptr, *jv = nullptr, *c = nullptr, *c2 = nullptr, *pack = nullptr,
           *rs = nullptr;
    int *info = nullptr;
    Pinned host, hrs;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    u64 seed = 0x5BD1A6ull;
    bool dist = false;  // partitioned context: vectors are this rank's rows, dots are all-reduced
    i64 goff = 0;       // global index of local element 0

    int AR(double *p, int cnt) { return dist ? sbd_dist_allreduce_internal(ctx, p, cnt, 0) : SBD_OK; }
    int sigma(const double *x, double *y) { return dist ? sbd_sigma_dist(ctx, x, y) : sbd_sigma(ctx, x, y); }

    ~Solver() {
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }

    double *vec(double *base, int i) const { return base + (i64)i * ld; }

    int readback(const double *src, int cnt, double *dst) {
        SBD_CUDA(ctx, cudaMemcpyAsync(dst, src, sizeof(double) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
        SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        return dist ? sbd_dist_check_internal(ctx) : SBD_OK;
    }

    const double *dg = nullptr;  // diagonal used by the preconditioner

    int setup(const double *x0, const double *diag_in) {
        // sizes and device buffers
        ld = std::max<i64>(32, (n + 31) / 32 * 32);
        SBD_CUDA(ctx, vw.ensure(sizeof(double) * (size_t)ld * (2 * (size_t)kmax + m)));
        V = vw.as<double>();
        W = V + (i64)kmax * ld;
        Tv = W + (i64)kmax * ld;
        const size_t n_aux = 2 * 144 + 1 + 2 * (size_t)kmax * kmax + 2 * (size_t)kmax * kMaxRoots + kMaxRoots + kmax +
                             (size_t)kmax * kmax + 2 * kMaxK + 2 * kMaxK + 32 + (size_t)kmax * kmax + kmax + 8;
        SBD_CUDA(ctx, aux.ensure(sizeof(double) * n_aux));
        SBD_CUDA(ctx, cudaMemsetAsync(aux.p, 0, sizeof(double) * n_aux, ctx->stream));
        double *p = aux.as<double>();
        auto take = [&](size_t cnt) {
            double *r = p;
            p += cnt;
            return r;
        };
        small = take(144);
        small2 = take(144);
        scale = take(1);
        T = take((size_t)kmax * kmax);
        G = take((size_t)kmax * kmax);
        Y = take((size_t)kmax * kMaxRoots);
        Yk = take((size_t)kmax * kMaxRoots);
        th = take(kMaxRoots);
        jw = take(kmax);
        jv = take((size_t)kmax * kmax);
        c = take(kMaxK);
        c2 = take(kMaxK);
        pack = take(2 * kMaxK + 32);
        rs = take((size_t)kmax * kmax + kmax);
        info = reinterpret_cast<int *>(take(8));
        SBD_CUDA(ctx, cudaMallocHost(&host.p, sizeof(double) * (2 * kMaxK + 32 + (size_t)3 * kmax * kmax + 2 * kmax)));
        SBD_CUDA(ctx, cudaMallocHost(&hrs.p, sizeof(double) * ((size_t)kmax * kmax + kmax)));
        SBD_CUDA(ctx, cudaEventCreate(&ev0));
        SBD_CUDA(ctx, cudaEventCreate(&ev1));
        if (diag_in) {
            dg = diag_in;
        } else {
            SBD_CUDA(ctx, diag.ensure(sizeof(double) * (size_t)n));
            if (int rc = sbd_diag(ctx, diag.as<double>())) return rc;
            dg = diag.as<double>();
        }

        // start vector (davidson.py:219-227)
        if (!x0) {
            const int nb = (int)std::min<i64>(grid_for(n, kArgBlock), 2 * (i64)ctx->num_sms);
            SBD_CUDA(ctx, part.ensure((sizeof(double) + sizeof(i64)) * nb));
            SBD_CUDA(ctx, cudaMemsetAsync(V, 0, sizeof(double) * n, ctx->stream));
            double *pv = part.as<double>();
            i64 *pi = reinterpret_cast<i64 *>(pv + nb);
            argmin_partial_kernel<<<nb, kArgBlock, 0, ctx->stream>>>(dg, n, pv, pi);
            if (!dist) {
                argmin_final_kernel<<<1, kArgBlock, 0, ctx->stream>>>(pv, pi, nb, n, V);
            } else {  // global argmin over the ranks: min value, then the smallest index holding it
                argmin_local_kernel<<<1, kArgBlock, 0, ctx->stream>>>(pv, pi, nb, n, goff, small);
                if (int rc = sbd_dist_allreduce_internal(ctx, small + 2, 1, 2)) return rc;
                argmin_candidate_kernel<<<1, 1, 0, ctx->stream>>>(small);
                if (int rc = sbd_dist_allreduce_internal(ctx, small + 3, 1, 2)) return rc;
                argmin_set_kernel<<<1, 1, 0, ctx->stream>>>(small, n, goff, V);
            }
            SBD_LAUNCHED(ctx, "davidson start vector");
        } else {
            if (int rc = sbd_vdots(ctx, x0, 1, ld, n, x0, small)) return rc;
            if (int rc = AR(small, 1)) return rc;
            if (int rc = readback(small, 1, host.p)) return rc;
            const double nrm = std::sqrt(std::max(host.p[0], 0.0));
            if (!(nrm > 0.0) || !std::isfinite(nrm)) return sbd_fail(ctx, SBD_EINVAL, "x0 must be nonzero and finite");
            set_scalar_kernel<<<1, 1, 0, ctx->stream>>>(scale, 1.0 / nrm);
            SBD_LAUNCHED(ctx, "davidson x0 scale");
            if (int rc = sbd_scale_copy(ctx, x0, V, n, scale)) return rc;
        }
        return SBD_OK;
    }

    // CGS2 of t against V[:k] given c = V^T t on the device; writes V[k] on success
    // (reference orthogonalize, davidson.py:166-185).  pre = pass-1 outputs already read back.
    int orthogonalize(int k, double *t, double t_norm2, const double *pre_c2, double pre_n2p, bool *ok) {
        *ok = false;
        const double norm0 = std::sqrt(std::max(t_norm2, 0.0));
        if (norm0 == 0.0) return SBD_OK;
        double *hb = host.p;
        if (o.reorthogonalize) {
            double n2p;
            std::vector<double> c2h(k);
            if (!pre_c2) {
                if (int rc = sbd_gs_update(ctx, V, k, ld, n, c, t, small2)) return rc;
                if (int rc = AR(small2, k + 1)) return rc;
                if (int rc = readback(small2, k + 1, hb)) return rc;
                std::memcpy(c2h.data(), hb, sizeof(double) * k);
                n2p = hb[k];
            } else {
                std::memcpy(c2h.data(), pre_c2, sizeof(double) * k);
                n2p = pre_n2p;
            }
            if (o.selective_reorth && n2p >= 0.5 * t_norm2) {  // |t1| >= |t0| / sqrt(2): one pass is enough
                const double norm = std::sqrt(std::max(n2p, 0.0));
                if (norm < 1e-12 * norm0 || norm == 0.0) return SBD_OK;
                set_scalar_kernel<<<1, 1, 0, ctx->stream>>>(scale, 1.0 / norm);
                SBD_LAUNCHED(ctx, "davidson scale");
                if (int rc = sbd_scale_copy(ctx, t, vec(V, k), n, scale)) return rc;
                *ok = true;
                return SBD_OK;
            }
            double cc = 0.0;
            for (int i = 0; i < k; ++i) cc += c2h[i] * c2h[i];
            const double n2 = n2p - cc;  // |t' - V c2|^2 for orthonormal V
            copy_small_kernel<<<1, kMaxK, 0, ctx->stream>>>(small2, c2, k);
            SBD_LAUNCHED(ctx, "davidson c2");
            if (n2p > 0.0 && n2 > 0.5 * n2p) {
                if (std::sqrt(n2) < 1e-12 * norm0) return SBD_OK;
                set_scalar_kernel<<<1, 1, 0, ctx->stream>>>(scale, 1.0 / std::sqrt(n2));
                SBD_LAUNCHED(ctx, "davidson scale");
                if (int rc = sbd_gs_finalize(ctx, V, k, ld, n, c2, t, vec(V, k), scale, small2)) return rc;
                *ok = true;
                return SBD_OK;
            }
            if (int rc = sbd_gs_update_nodots(ctx, V, k, ld, n, c2, t, small2)) return rc;
        } else {
            if (int rc = sbd_gs_update_nodots(ctx, V, k, ld, n, c, t, small2)) return rc;
        }
        if (int rc = AR(small2, 1)) return rc;
        if (int rc = readback(small2, 1, hb)) return rc;
        const double norm = std::sqrt(std::max(hb[0], 0.0));
        if (norm < 1e-12 * norm0 || norm == 0.0) return SBD_OK;
        set_scalar_kernel<<<1, 1, 0, ctx->stream>>>(scale, 1.0 / norm);
        SBD_LAUNCHED(ctx, "davidson scale");
        if (int rc = sbd_scale_copy(ctx, t, vec(V, k), n, scale)) return rc;
        *ok = true;
        return SBD_OK;
    }

    // c = V^T t and |t|^2 for a fresh direction t (one extra pass)
    int project(int k, double *t, double *t_norm2) {
        if (int rc = sbd_vdots2(ctx, V, k, ld, n, t, t, small)) return rc;
        if (int rc = AR(small, k)) return rc;
        copy_small_kernel<<<1, kMaxK, 0, ctx->stream>>>(small, c, k);
        SBD_LAUNCHED(ctx, "davidson c");
        if (int rc = sbd_vdots(ctx, t, 1, ld, n, t, small + 2 * kMaxK)) return rc;
        if (int rc = AR(small + 2 * kMaxK, 1)) return rc;
        if (int rc = readback(small + 2 * kMaxK, 1, host.p)) return rc;
        *t_norm2 = host.p[0];
        return SBD_OK;
    }

    int run(const double *diag_in, const double *x0, double *evals, double *res_out, double *evecs, i64 ldu,
            sbd_davidson_stats *st) {
        if (int rc = setup(x0, diag_in)) return rc;
        int k = 1, mk = 1, jp = 0;
        bool ritz_rotated = false;
        std::vector<double> theta(m, 0.0), res(m, INFINITY);
        double sigma_ms = 0.0;
        for (int iteration = 1; iteration <= o.max_iters; ++iteration) {
            SbdRange range("sbd/davidson_iteration");
            const auto t_iter = std::chrono::steady_clock::now();
            auto iter_done = [&]() {
                if (st->iter_ms_hist)
                    st->iter_ms_hist[iteration - 1] =
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_iter).count();
            };
            st->iterations = iteration;
            SBD_CUDA(ctx, cudaEventRecord(ev0, ctx->stream));
            if (int rc = sigma(vec(V, k - 1), vec(W, k - 1))) return rc;
            SBD_CUDA(ctx, cudaEventRecord(ev1, ctx->stream));
            st->n_applies++;

            // T[:, k-1] = V^T w and the Gram row of v_{k-1}: one pass over V
            if (int rc = sbd_vdots2(ctx, V, k, ld, n, vec(W, k - 1), vec(V, k - 1), small)) return rc;
            if (int rc = AR(small, 2 * k)) return rc;
            set_tg_kernel<<<1, kMaxK, 0, ctx->stream>>>(T, G, small, k, kmax);
            SBD_LAUNCHED(ctx, "davidson T");
            // Rayleigh-Ritz in place on T (davidson.py:251)
            if (int rc = sbd_jacobi(ctx, T, k, kmax, jw, jv, kMaxSweeps, info)) return rc;
            mk = std::min(m, k);
            ritz_prep_kernel<<<1, 256, 0, ctx->stream>>>(jv, jw, k, mk, Y, th);
            SBD_LAUNCHED(ctx, "davidson ritz");
            ritz_rotated = false;

            // residuals, preconditioned corrections and V^T t in one pass
            jp = std::min(jp, mk - 1);
            if (int rc = sbd_residual_precond_target(ctx, V, W, k, ld, n, Y, th, mk, jp, dg,
                                                     o.precond_delta, Tv, ld, small))
                return rc;
            if (int rc = AR(small, k + 1 + mk)) return rc;
            copy_small_kernel<<<1, kMaxK, 0, ctx->stream>>>(small, c, k);
            SBD_LAUNCHED(ctx, "davidson c");
            // speculative CGS pass 1 on the projected root, read back with the pack
            const bool spec = o.reorthogonalize && k < kmax && iteration < o.max_iters;
            if (spec) {
                if (int rc = sbd_gs_update(ctx, V, k, ld, n, c, vec(Tv, jp), small2)) return rc;
                if (int rc = AR(small2, k + 1)) return rc;
            }
            pack_kernel<<<1, 256, 0, ctx->stream>>>(jw, small, small2, info, G, kmax, k, mk, o.track_orthogonality,
                                                   spec ? 1 : 0, pack);
            SBD_LAUNCHED(ctx, "davidson pack");
            const int npk = 2 * mk + 3;
            double *hv = host.p;
            if (int rc = readback(pack, npk + (spec ? k + 1 : 0), hv)) return rc;
            float ms = 0.f;
            SBD_CUDA(ctx, cudaEventElapsedTime(&ms, ev0, ev1));
            sigma_ms += ms;
            if (hv[2 * mk + 1] >= kMaxSweeps) return sbd_fail(ctx, SBD_ECUDA, "Jacobi sweep limit 64 reached without convergence");
            bool all_conv = true;
            int target = -1;
            for (int j = 0; j < mk; ++j) {
                theta[j] = hv[j];
                res[j] = std::sqrt(std::max(hv[mk + j], 0.0));
                if (!(res[j] <= o.tol_residual)) {
                    all_conv = false;
                    if (target < 0) target = j;
                }
            }
            double t_norm2 = hv[2 * mk];
            const i64 it0 = (i64)(iteration - 1);
            if (st->theta_hist)
                for (int j = 0; j < m; ++j) st->theta_hist[it0 * m + j] = j < mk ? theta[j] : NAN;
            if (st->res_hist)
                for (int j = 0; j < m; ++j) st->res_hist[it0 * m + j] = j < mk ? res[j] : NAN;
            if (st->ortho_hist) st->ortho_hist[it0] = o.track_orthogonality ? hv[2 * mk + 2] : NAN;
            if (st->apply_ms_hist) st->apply_ms_hist[it0] = ms;

            if (all_conv) {
                st->converged = 1;
                iter_done();
                break;
            }
            if (iteration == o.max_iters) {
                iter_done();
                break;
            }

            double *t = vec(Tv, target);
            std::vector<double> pre_c2;
            double pre_n2p = 0.0;
            if (spec && target == jp) {
                pre_c2.assign(hv + npk, hv + npk + k);
                pre_n2p = hv[npk + k];
            }
            if (target != jp) {  // the fused projection used another root: one extra pass
                if (int rc = project(k, t, &t_norm2)) return rc;
                jp = target;
            }

            if (k == kmax) {
                // thick restart (davidson.py:280-289): rotate V and W in place
                cols_kernel<<<1, 256, 0, ctx->stream>>>(jv, k, keep, Yk);
                SBD_LAUNCHED(ctx, "davidson restart Y");
                if (int rc = sbd_rotate(ctx, V, k, ld, n, Yk, keep)) return rc;
                if (int rc = sbd_rotate(ctx, W, k, ld, n, Yk, keep)) return rc;
                // keep x keep bookkeeping on the host: G' = Yk^T G Yk, c' = Yk^T c
                double *hy = host.p + 2 * kMaxK + 32, *hg = hy + (size_t)kmax * kmax, *hc = hg + (size_t)kmax * kmax;
                SBD_CUDA(ctx, cudaMemcpyAsync(hy, jv, sizeof(double) * k * k, cudaMemcpyDeviceToHost, ctx->stream));
                SBD_CUDA(ctx, cudaMemcpyAsync(hg, G, sizeof(double) * kmax * kmax, cudaMemcpyDeviceToHost, ctx->stream));
                SBD_CUDA(ctx, cudaMemcpyAsync(hc, c, sizeof(double) * k, cudaMemcpyDeviceToHost, ctx->stream));
                SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
                std::vector<double> gy((size_t)k * keep, 0.0);  // G Yk
                for (int i = 0; i < k; ++i)
                    for (int l = 0; l < k; ++l) {
                        const double g = hg[(size_t)i * kmax + l];
                        for (int j = 0; j < keep; ++j) gy[(size_t)i * keep + j] += g * hy[(size_t)l * k + j];
                    }
                for (int a = 0; a < keep; ++a) {
                    for (int b = 0; b < keep; ++b) {
                        double s = 0.0;
                        for (int i = 0; i < k; ++i) s += hy[(size_t)i * k + a] * gy[(size_t)i * keep + b];
                        hrs.p[a * keep + b] = s;
                    }
                    double s = 0.0;
                    for (int i = 0; i < k; ++i) s += hy[(size_t)i * k + a] * hc[i];
                    hrs.p[keep * keep + a] = s;
                }
                SBD_CUDA(ctx, cudaMemcpyAsync(rs, hrs.p, sizeof(double) * (keep * keep + keep), cudaMemcpyHostToDevice,
                                              ctx->stream));
                restart_kernel<<<1, 256, 0, ctx->stream>>>(T, G, kmax, jw, rs, keep, c);
                SBD_LAUNCHED(ctx, "davidson restart");
                if (st->restart_iters && st->restarts < o.max_iters) st->restart_iters[st->restarts] = iteration;
                st->restarts++;
                k = keep;
                ritz_rotated = true;
            }

            bool ok = false;
            if (int rc = orthogonalize(k, t, t_norm2, pre_c2.empty() ? nullptr : pre_c2.data(), pre_n2p, &ok))
                return rc;
            for (int attempts = 0; !ok && attempts < 3; ++attempts) {
                st->breakdowns++;
                random_normal_kernel<<<2 * ctx->num_sms, 256, 0, ctx->stream>>>(t, n, goff, seed + 0x1000ull * st->breakdowns);
                SBD_LAUNCHED(ctx, "davidson random direction");
                double nn = 0.0;
                if (int rc = project(k, t, &nn)) return rc;
                if (int rc = orthogonalize(k, t, nn, nullptr, 0.0, &ok)) return rc;
            }
            iter_done();
            if (!ok) break;
            ++k;
        }

        // Ritz vectors of the last Rayleigh-Ritz (davidson.py:256), computed once
        if (evecs) {
            if (ritz_rotated) {
                std::vector<double> yr((size_t)k * mk, 0.0);
                for (int j = 0; j < mk; ++j) yr[(size_t)j * mk + j] = 1.0;
                std::memcpy(hrs.p, yr.data(), sizeof(double) * yr.size());
                SBD_CUDA(ctx, cudaMemcpyAsync(Y, hrs.p, sizeof(double) * yr.size(), cudaMemcpyHostToDevice, ctx->stream));
            }  // else Y already holds evecs[:, :mk] of this k
            if (int rc = sbd_combine(ctx, V, k, ld, n, Y, mk, evecs, ldu)) return rc;
        }
        SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        for (int j = 0; j < m; ++j) {
            if (evals) evals[j] = j < mk ? theta[j] : NAN;
            if (res_out) res_out[j] = j < mk ? res[j] : NAN;
        }
        st->n_found = mk;
        st->sigma_ms = sigma_ms;
        return SBD_OK;
    }
};

}  // namespace

extern "C" {

int sbd_davidson_default_opts(sbd_davidson_opts *o) {
    if (!o) return sbd_fail(nullptr, SBD_EINVAL, "null options");
    o->n_roots = 1;
    o->tol_residual = 1e-8;
    o->max_iters = 200;
    o->max_subspace = 32;
    o->restart_keep = 4;
    o->precond_delta = 1e-6;
    o->reorthogonalize = 1;
    o->track_orthogonality = 1;
    o->selective_reorth = 0;
    return SBD_OK;
}

int sbd_davidson(sbd_ctx *ctx, const sbd_davidson_opts *opts, const double *diag_dev, const double *x0_dev,
                 double *evals_host,
                 double *res_norms_host, double *evecs_dev, int64_t ldu, sbd_davidson_stats *stats) {
    SBD_CHECK_CTX(ctx);
    if (!opts) return sbd_fail(ctx, SBD_EINVAL, "null options");
    const sbd_davidson_opts &o = *opts;
    // option validation as DavidsonOptions (davidson.py:42-53) plus the device limits
    if (!(1 <= o.n_roots && o.n_roots <= o.restart_keep && o.restart_keep <= o.max_subspace))
        return sbd_fail(ctx, SBD_EINVAL, "need 1 <= n_roots <= restart_keep <= max_subspace");
    if (!(o.tol_residual > 0)) return sbd_fail(ctx, SBD_EINVAL, "tol_residual must be positive");
    if (!(o.precond_delta > 0)) return sbd_fail(ctx, SBD_EINVAL, "precond_delta must be positive");
    if (o.max_iters < 1) return sbd_fail(ctx, SBD_EINVAL, "max_iters must be at least 1");
    if (o.max_subspace > kMaxK) return sbd_fail(ctx, SBD_EINVAL, "max_subspace must be <= 64 on the B200 path");
    if (o.n_roots > kMaxRoots) return sbd_fail(ctx, SBD_EINVAL, "n_roots must be <= 8 on the B200 path");
    if (!ctx->have_integrals || !ctx->sec[0].present || !ctx->sec[1].present)
        return sbd_fail(ctx, SBD_EINVAL, "integrals and strings must be set first");
    i64 n, nglob;
    const bool dist = ctx->dist.on && ctx->dist.nranks > 1;
    if (ctx->explicit_mode) {
        n = nglob = ctx->n_det;
    } else {
        // a partitioned context (sbd_dist_init) solves over its own rows, all-reducing every dot product
        if (!dist && ctx->own_rows() != ctx->sec[0].n)
            return sbd_fail(ctx, SBD_EINVAL, "sbd_davidson: a row-windowed context must be partitioned (sbd_dist_init)");
        n = ctx->own_rows() * ctx->sec[1].n;
        nglob = ctx->sec[0].n * ctx->sec[1].n;
    }
    if (nglob < 1) return sbd_fail(ctx, SBD_EINVAL, "empty problem");
    if (nglob < o.n_roots) return sbd_fail(ctx, SBD_EINVAL, "cannot extract n_roots roots from this dimension");
    sbd_davidson_stats local;
    std::memset(&local, 0, sizeof(local));
    sbd_davidson_stats *st = stats ? stats : &local;
    st->iterations = st->converged = st->n_applies = st->restarts = st->breakdowns = st->n_found = 0;
    st->sigma_ms = 0.0;
    Solver s;
    s.ctx = ctx;
    s.o = o;
    s.n = n;
    s.dist = dist;
    s.goff = dist ? ctx->own_lo() * ctx->sec[1].n : 0;
    s.m = o.n_roots;
    s.kmax = (int)std::min<i64>(o.max_subspace, nglob);
    s.keep = std::min(o.restart_keep, s.kmax);
    return s.run(diag_dev, x0_dev, evals_host, res_norms_host, evecs_dev, ldu > 0 ? ldu : n, st);
}

}  // extern "C"
