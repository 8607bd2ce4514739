// Same-spin parts of sigma as dense fp64 GEMMs, for dense string sets.
//
// Reference: the beta singles/doubles (task 1) and alpha singles/doubles (task 2) of
// _product_row (apply.py:217-233).  With A (B) the alpha (beta) same-spin connection
// matrix, sigma gets A X + X B^T plus the spectator-dependent part of the singles:
//   single i -> j over orbital pair P with phase s:  s (F + J[P][spectator]) x
// (sbd_excite.cu: Conn.c = s F, J tables per pair and spectator string).
// When a sector's strings are a large fraction of the string space (cfg1, the full
// 12-orbital set: 261 in-set connections per string, 28% of the row), streaming a 2 KB
// segment per connection (the side kernels) moves 8 c-bar bytes per determinant while the
// dense product is 2 n flops per determinant on the fp64 tensor pipe.  This file builds,
// per sector, the dense matrix of the spectator-independent coefficients (doubles, and
// s F of the singles) and a singles-only connection list whose coefficient is 0, so the
// side kernels keep streaming just the s J[P][spectator] term (36 of 261 connections at
// cfg1), and adds A X + X B^T with cuBLAS DGEMM (a plain library GEMM: two 924^3
// products at cfg1), on an auxiliary stream concurrent with the beta stream and task 0.
#include <cublas_v2.h>

#include <cstdlib>

#include "sbd_internal.cuh"

namespace {

// dense[i][tgt] = c for every connection of string i (doubles: the element; singles: s F)
__global__ void dense_fill_kernel(i64 n, const int64_t *__restrict__ off, const Conn *__restrict__ conn,
                                  double *__restrict__ dense) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (i64 e = off[i]; e < off[i + 1]; ++e) dense[i * n + conn[e].tgt] = conn[e].c;
}

// singles of each string (the first s_off[i+1] - s_off[i] connections of its row) with c = 0
__global__ void singles_j_kernel(i64 n, const int64_t *__restrict__ off, const int64_t *__restrict__ s_off,
                                 const Conn *__restrict__ conn, Conn *__restrict__ out) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const i64 ns = s_off[i + 1] - s_off[i];
    for (i64 k = 0; k < ns; ++k) {
        Conn c = conn[off[i] + k];
        c.c = 0.0;
        out[s_off[i] + k] = c;
    }
}

constexpr i64 kGemmMaxStrings = 6144;  // dense matrices up to 288 MB per sector

}  // namespace

bool sbd_samespin_gemm_on(const sbd_ctx *ctx) {
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    if (ctx->explicit_mode || (ctx->dist.on && ctx->dist.nranks > 1) || !A.built || !B.built) return false;
    const char *e = getenv("SBD_DENSE_GEMM");
    if (e && e[0] == '0') return false;
    if (A.n == 0 || B.n == 0 || A.n > kGemmMaxStrings || B.n > kGemmMaxStrings) return false;
    if (e && e[0] == '1') return true;
    // streaming 8 c-bar bytes from L2 vs 2 n flops on the DMMA pipe per determinant: dense wins above
    // ~1/7 of the row; both sectors (the alpha and the beta products run together), and only where the
    // products are worth a cuBLAS launch and a second stream (n >= 256)
    auto dense = [](const Sector &S) { return S.n >= 256 && 8 * (S.ns + S.nd) >= S.n * S.n; };
    return dense(A) && dense(B);
}

int sbd_samespin_gemm_prepare(sbd_ctx *ctx) {
    if (ctx->ssg_valid) return SBD_OK;
    cudaStream_t st = ctx->stream;
    for (int spin = 0; spin < 2; ++spin) {
        Sector &S = ctx->sec[spin];
        SBD_CUDA(ctx, S.dense.ensure(sizeof(double) * S.n * S.n));
        SBD_CUDA(ctx, cudaMemsetAsync(S.dense.p, 0, sizeof(double) * S.n * S.n, st));
        dense_fill_kernel<<<grid_for(S.n, 128), 128, 0, st>>>(S.n, S.conn_off.as<int64_t>(), S.conn.as<Conn>(),
                                                             S.dense.as<double>());
        SBD_CUDA(ctx, S.conn_j.ensure(sizeof(Conn) * (S.ns + 1)));
        singles_j_kernel<<<grid_for(S.n, 128), 128, 0, st>>>(S.n, S.conn_off.as<int64_t>(), S.s_off.as<int64_t>(),
                                                            S.conn.as<Conn>(), S.conn_j.as<Conn>());
        SBD_LAUNCHED(ctx, "same-spin dense matrices");
    }
    if (!ctx->cublas) {
        cublasHandle_t h;
        if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return sbd_fail(ctx, SBD_ECUDA, "cublasCreate failed");
        ctx->cublas = h;
    }
    ctx->ssg_valid = true;
    return SBD_OK;
}

__global__ void add_kernel(double *__restrict__ y, const double *__restrict__ z, i64 n) {
    const i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] += z[i];
}

// Z = A[own rows, :] X + X[own rows] B^T on the auxiliary stream (row-major Z, X; column-major
// cuBLAS views: Z^T (nb x rows) = X^T A^T[:, own] + B X^T[:, own]), started once x is complete so the
// two DGEMMs share the SMs with the beta stream and task 0 instead of following the alpha side.
int sbd_samespin_gemm_start(sbd_ctx *ctx, const double *x_full) {
    const Sector &A = ctx->sec[0], &B = ctx->sec[1];
    const i64 na = A.n, nb = B.n, lo = ctx->own_lo(), rows = ctx->own_rows();
    if (rows <= 0) return SBD_OK;
    if (!ctx->aux_stream) SBD_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
    if (!ctx->aux_ev[0]) {
        for (auto &e : ctx->aux_ev) SBD_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    SBD_CUDA(ctx, ctx->ssg_z.ensure(sizeof(double) * rows * nb));
    SBD_CUDA(ctx, cudaEventRecord(ctx->aux_ev[0], ctx->stream));
    SBD_CUDA(ctx, cudaStreamWaitEvent(ctx->aux_stream, ctx->aux_ev[0], 0));
    cublasHandle_t h = static_cast<cublasHandle_t>(ctx->cublas);
    if (cublasSetStream(h, ctx->aux_stream) != CUBLAS_STATUS_SUCCESS) return sbd_fail(ctx, SBD_ECUDA, "cublasSetStream");
    const double one = 1.0, zero = 0.0;
    double *z = ctx->ssg_z.as<double>();
    if (cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)nb, (int)rows, (int)na, &one, x_full, (int)nb,
                    A.dense.as<double>() + lo * na, (int)na, &zero, z, (int)nb) != CUBLAS_STATUS_SUCCESS)
        return sbd_fail(ctx, SBD_ECUDA, "cublasDgemm (alpha)");
    if (cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)nb, (int)rows, (int)nb, &one, B.dense.as<double>(), (int)nb,
                    x_full + lo * nb, (int)nb, &one, z, (int)nb) != CUBLAS_STATUS_SUCCESS)
        return sbd_fail(ctx, SBD_ECUDA, "cublasDgemm (beta)");
    return SBD_OK;
}

// everything queued on the auxiliary stream so far is what finish() waits for
int sbd_samespin_gemm_mark(sbd_ctx *ctx) {
    SBD_CUDA(ctx, cudaEventRecord(ctx->aux_ev[1], ctx->aux_stream));
    return SBD_OK;
}

// y[own rows] += Z, after the alpha side (which writes y)
int sbd_samespin_gemm_finish(sbd_ctx *ctx, double *y) {
    const i64 n = ctx->own_rows() * ctx->sec[1].n;
    if (n <= 0) return SBD_OK;
    SBD_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0));
    add_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(y, ctx->ssg_z.as<double>(), n);
    SBD_LAUNCHED(ctx, "same-spin dense add");
    return SBD_OK;
}

void sbd_samespin_gemm_release(sbd_ctx *ctx) {
    if (ctx->cublas) cublasDestroy(static_cast<cublasHandle_t>(ctx->cublas));
    ctx->cublas = nullptr;
    if (ctx->aux_stream) {
        cudaStreamSynchronize(ctx->aux_stream);
        cudaStreamDestroy(ctx->aux_stream);
    }
    ctx->aux_stream = nullptr;
    for (auto &e : ctx->aux_ev)
        if (e) cudaEventDestroy(e);
}
