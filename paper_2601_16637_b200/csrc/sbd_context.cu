// Context lifetime, uploads, table export and error plumbing of the C ABI.
#include <cstring>
#include <new>

#include "sbd_internal.cuh"

static thread_local std::string g_last_error;

void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

cudaError_t DevBuf::ensure(size_t nbytes) {
    if (nbytes <= bytes && p) return cudaSuccess;
    release();
    if (nbytes == 0) nbytes = 16;
    cudaError_t e = cudaMalloc(&p, nbytes);
    if (e == cudaSuccess) bytes = nbytes;
    else p = nullptr;
    return e;
}

int sbd_fail(sbd_ctx *ctx, int code, const std::string &msg) {
    g_last_error = msg;
    if (ctx) ctx->err = msg;
    return code;
}

int sbd_cuda_fail(sbd_ctx *ctx, cudaError_t e, const char *where) {
    std::string m = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return sbd_fail(ctx, SBD_ECUDA, m);
}

template <class T>
static int copy_down(sbd_ctx *ctx, T *dst, const DevBuf &src, i64 count) {
    if (!dst || count == 0) return SBD_OK;
    SBD_CUDA(ctx, cudaMemcpy(dst, src.p, sizeof(T) * count, cudaMemcpyDeviceToHost));
    return SBD_OK;
}

static int copy_down_i32_to_i64(sbd_ctx *ctx, int64_t *dst, const DevBuf &src, i64 count) {
    if (!dst || count == 0) return SBD_OK;
    std::vector<int32_t> tmp(count);
    SBD_CUDA(ctx, cudaMemcpy(tmp.data(), src.p, sizeof(int32_t) * count, cudaMemcpyDeviceToHost));
    for (i64 i = 0; i < count; ++i) dst[i] = tmp[i];
    return SBD_OK;
}

extern "C" {

int sbd_abi_version(void) { return 1; }

const char *sbd_last_error(const sbd_ctx *ctx) {
    if (ctx && !ctx->err.empty()) return ctx->err.c_str();
    return g_last_error.c_str();
}

int sbd_create(int device, sbd_ctx **out) {
    if (!out) return sbd_fail(nullptr, SBD_EINVAL, "sbd_create: out is NULL");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return sbd_cuda_fail(nullptr, e, "cudaGetDeviceCount");
    if (device < 0 || device >= ndev)
        return sbd_fail(nullptr, SBD_EINVAL, "sbd_create: device " + std::to_string(device) + " not present");
    e = cudaSetDevice(device);
    if (e != cudaSuccess) return sbd_cuda_fail(nullptr, e, "cudaSetDevice");
    sbd_ctx *ctx = new (std::nothrow) sbd_ctx();
    if (!ctx) return sbd_fail(nullptr, SBD_ECUDA, "sbd_create: out of host memory");
    ctx->device = device;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
        ctx->num_sms = sms;
    *out = ctx;
    return SBD_OK;
}

int sbd_destroy(sbd_ctx *ctx) {
    if (!ctx) return SBD_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
    }
    for (cudaEvent_t e : ctx->events) cudaEventDestroy(e);
    sbd_dist_release(ctx);
    sbd_samespin_gemm_release(ctx);
    delete ctx;
    return SBD_OK;
}

int sbd_set_stream(sbd_ctx *ctx, void *stream) {
    SBD_CHECK_CTX(ctx);
    ctx->stream = reinterpret_cast<cudaStream_t>(stream);
    return SBD_OK;
}

int sbd_set_integrals(sbd_ctx *ctx, int norb, const double *h_host, const double *eri_host, int64_t n_eri,
                      double e_core) {
    SBD_CHECK_CTX(ctx);
    if (norb < 1 || norb > 64) return sbd_fail(ctx, SBD_EINVAL, "norb must be in [1, 64]");
    i64 npair = (i64)norb * (norb + 1) / 2;
    if (n_eri != npair * (npair + 1) / 2)
        return sbd_fail(ctx, SBD_EINVAL, "eri length " + std::to_string(n_eri) + " != npair*(npair+1)/2 = " +
                                             std::to_string(npair * (npair + 1) / 2));
    if (!h_host || !eri_host) return sbd_fail(ctx, SBD_EINVAL, "null integral pointer");
    ctx->norb = norb;
    ctx->npair = npair;
    ctx->n_eri = n_eri;
    ctx->e_core = e_core;
    SBD_CUDA(ctx, ctx->h.ensure(sizeof(double) * norb * norb));
    SBD_CUDA(ctx, ctx->eri.ensure(sizeof(double) * n_eri));
    SBD_CUDA(ctx, ctx->dpq.ensure(sizeof(double) * norb * norb));
    std::vector<double> dpq((size_t)norb * norb);
    for (int p = 0; p < norb; ++p)
        for (int q = 0; q < norb; ++q) dpq[(size_t)p * norb + q] = eri_host[tri_idx(tri_idx(p, p), tri_idx(q, q))];
    SBD_CUDA(ctx, cudaMemcpy(ctx->h.p, h_host, sizeof(double) * norb * norb, cudaMemcpyHostToDevice));
    SBD_CUDA(ctx, cudaMemcpy(ctx->eri.p, eri_host, sizeof(double) * n_eri, cudaMemcpyHostToDevice));
    SBD_CUDA(ctx, cudaMemcpy(ctx->dpq.p, dpq.data(), sizeof(double) * norb * norb, cudaMemcpyHostToDevice));
    ctx->ld_vpp = (npair + 1) / 2 * 2;
    {
        const i64 ld = ctx->ld_vpp;
        std::vector<double> vpp((size_t)npair * 4 * ld, 0.0);
        for (i64 P = 0; P < npair; ++P)
            for (int sa = 0; sa < 2; ++sa)
                for (i64 Q = 0; Q < npair; ++Q) {
                    const double v = eri_host[tri_idx(P, Q)];
                    vpp[(size_t)(2 * P + sa) * 2 * ld + Q] = sa ? -v : v;
                    vpp[(size_t)(2 * P + sa) * 2 * ld + ld + Q] = sa ? v : -v;
                }
        SBD_CUDA(ctx, ctx->vpp.ensure(sizeof(double) * vpp.size()));
        SBD_CUDA(ctx, cudaMemcpy(ctx->vpp.p, vpp.data(), sizeof(double) * vpp.size(), cudaMemcpyHostToDevice));
    }
    ctx->have_integrals = true;
    ctx->sec[0].built = ctx->sec[1].built = false;
    ctx->diag_valid = false;
    return SBD_OK;
}

int sbd_set_strings(sbd_ctx *ctx, int spin, const uint64_t *strings, int64_t n, int n_elec) {
    SBD_CHECK_CTX(ctx);
    if (spin != 0 && spin != 1) return sbd_fail(ctx, SBD_EINVAL, "spin must be 0 (alpha) or 1 (beta)");
    if (!ctx->have_integrals) return sbd_fail(ctx, SBD_EINVAL, "set integrals before strings");
    if (n < 0 || (n > 0 && !strings)) return sbd_fail(ctx, SBD_EINVAL, "bad string array");
    if (n >= (i64)INT32_MAX) return sbd_fail(ctx, SBD_EINVAL, "too many strings for int32 indexing");
    const char *label = spin ? "beta" : "alpha";
    int norb = ctx->norb;
    for (i64 i = 0; i < n; ++i) {  // SelectedBasis._validate_strings, basis.py:185-194
        u64 s = strings[i];
        if (norb < 64 && (s >> norb)) {
            char buf[128];
            snprintf(buf, sizeof buf, "%s string %#llx has bits above orbital %d", label, (unsigned long long)s, norb - 1);
            return sbd_fail(ctx, SBD_EINVAL, buf);
        }
        if (__builtin_popcountll(s) != n_elec) {
            char buf[128];
            snprintf(buf, sizeof buf, "%s string %#llx has %d electrons, expected %d", label, (unsigned long long)s,
                     __builtin_popcountll(s), n_elec);
            return sbd_fail(ctx, SBD_EINVAL, buf);
        }
    }
    Sector &s = ctx->sec[spin];
    s.n = n;
    s.n_elec = n_elec;
    s.present = true;
    s.built = false;
    s.host.assign(strings, strings + n);
    SBD_CUDA(ctx, s.str.ensure(sizeof(u64) * (n ? n : 1)));
    if (n) SBD_CUDA(ctx, cudaMemcpy(s.str.p, strings, sizeof(u64) * n, cudaMemcpyHostToDevice));
    ctx->diag_valid = false;
    ctx->explicit_mode = false;  // sbd_set_dets re-enables it after setting both sectors
    if (spin == 0) ctx->row_lo = 0, ctx->row_hi = -1;
    return SBD_OK;
}

#ifdef SBD_TIMING
#include <chrono>
#include <cstdio>
#define SBD_TSTAMP(label)                                                                                   \
    do {                                                                                                    \
        cudaStreamSynchronize(ctx->stream);                                                                 \
        static auto t_prev = std::chrono::steady_clock::now();                                              \
        auto t_now = std::chrono::steady_clock::now();                                                      \
        fprintf(stderr, "[sbd timing] %s %.3f ms\n", label,                                                 \
                std::chrono::duration<double, std::milli>(t_now - t_prev).count());                          \
        t_prev = t_now;                                                                                     \
    } while (0)
#else
#define SBD_TSTAMP(label) \
    do {                  \
    } while (0)
#endif

int sbd_build_tables(sbd_ctx *ctx) {
    SBD_CHECK_CTX(ctx);
    SbdRange range("sbd/build_tables");
    if (!ctx->have_integrals) return sbd_fail(ctx, SBD_EINVAL, "integrals not set");
    SBD_TSTAMP("start");
    for (int spin = 0; spin < 2; ++spin) {
        Sector &s = ctx->sec[spin];
        if (!s.present) continue;
        int rc = sbd_sort_strings(ctx, s);
        if (rc) return rc;
        SBD_TSTAMP("sort");
        rc = sbd_build_sector_tables(ctx, s);
        if (rc) return rc;
        SBD_TSTAMP("excitation tables");
    }
    for (int spin = 0; spin < 2; ++spin) {
        Sector &s = ctx->sec[spin];
        if (!s.present) continue;
        // J tables need the OTHER sector's strings; a lone sector uses itself
        const Sector &o = ctx->sec[1 - spin].present ? ctx->sec[1 - spin] : s;
        int rc = sbd_build_coefficients(ctx, s, o);
        if (rc) return rc;
        SBD_TSTAMP("coefficients + J + SELL");
        s.built = true;
    }
    if (ctx->explicit_mode) {
        int rc = sbd_build_explicit_index(ctx);
        if (rc) return rc;
    }
    ctx->diag_valid = false;
    ctx->dci.valid = false;
    ctx->ssg_valid = false;
    ctx->dist.planned = false;  // the exchange plan is built from the alpha table
    SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SBD_OK;
}

int sbd_table_counts(sbd_ctx *ctx, int spin, int64_t *n_strings, int64_t *n_singles, int64_t *n_doubles) {
    SBD_CHECK_CTX(ctx);
    if (spin != 0 && spin != 1) return sbd_fail(ctx, SBD_EINVAL, "bad spin");
    const Sector &s = ctx->sec[spin];
    if (!s.built) return sbd_fail(ctx, SBD_EINVAL, "tables not built");
    if (n_strings) *n_strings = s.n;
    if (n_singles) *n_singles = s.ns;
    if (n_doubles) *n_doubles = s.nd;
    return SBD_OK;
}

static int export_sector(sbd_ctx *ctx, Sector &s, int64_t *s_off, int64_t *s_tgt, int16_t *s_hole, int16_t *s_part,
                         int8_t *s_phase, int64_t *d_off, int64_t *d_tgt, int16_t *d_h1, int16_t *d_h2, int16_t *d_p1,
                         int16_t *d_p2, int8_t *d_phase) {
    SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    int rc = 0;
    rc |= copy_down(ctx, s_off, s.s_off, s.n + 1);
    rc |= copy_down_i32_to_i64(ctx, s_tgt, s.s_tgt, s.ns);
    rc |= copy_down(ctx, s_hole, s.s_hole, s.ns);
    rc |= copy_down(ctx, s_part, s.s_part, s.ns);
    rc |= copy_down(ctx, s_phase, s.s_phase, s.ns);
    rc |= copy_down(ctx, d_off, s.d_off, s.n + 1);
    rc |= copy_down_i32_to_i64(ctx, d_tgt, s.d_tgt, s.nd);
    rc |= copy_down(ctx, d_h1, s.d_h1, s.nd);
    rc |= copy_down(ctx, d_h2, s.d_h2, s.nd);
    rc |= copy_down(ctx, d_p1, s.d_p1, s.nd);
    rc |= copy_down(ctx, d_p2, s.d_p2, s.nd);
    rc |= copy_down(ctx, d_phase, s.d_phase, s.nd);
    return rc ? SBD_ECUDA : SBD_OK;
}

int sbd_export_table(sbd_ctx *ctx, int spin, int64_t *s_off, int64_t *s_tgt, int16_t *s_hole, int16_t *s_part,
                     int8_t *s_phase, int64_t *d_off, int64_t *d_tgt, int16_t *d_h1, int16_t *d_h2, int16_t *d_p1,
                     int16_t *d_p2, int8_t *d_phase) {
    SBD_CHECK_CTX(ctx);
    if (spin != 0 && spin != 1) return sbd_fail(ctx, SBD_EINVAL, "bad spin");
    Sector &s = ctx->sec[spin];
    if (!s.built) return sbd_fail(ctx, SBD_EINVAL, "tables not built");
    return export_sector(ctx, s, s_off, s_tgt, s_hole, s_part, s_phase, d_off, d_tgt, d_h1, d_h2, d_p1, d_p2, d_phase);
}

int sbd_export_sorted(sbd_ctx *ctx, int spin, uint64_t *sorted_host, int64_t *perm_host) {
    SBD_CHECK_CTX(ctx);
    if (spin != 0 && spin != 1) return sbd_fail(ctx, SBD_EINVAL, "bad spin");
    Sector &s = ctx->sec[spin];
    if (!s.built) return sbd_fail(ctx, SBD_EINVAL, "tables not built");
    SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    int rc = copy_down(ctx, sorted_host, s.sorted, s.n);
    rc |= copy_down_i32_to_i64(ctx, perm_host, s.perm, s.n);
    return rc ? SBD_ECUDA : SBD_OK;
}

// 128-bit strings: basis.py:62-103 + 362-403 on two-word masks (the reference's table builder is
// width-agnostic; its integrals stop at 64 orbitals, integrals.py:67-68, so no sigma here).
int sbd_table128_build(sbd_ctx *ctx, int norb, const uint64_t *words, int64_t n, int n_elec) {
    SBD_CHECK_CTX(ctx);
    SbdRange range("sbd/table128_build");
    Sector &s = ctx->t128;
    s.built = false;
    if (norb < 1 || norb > 128) return sbd_fail(ctx, SBD_EINVAL, "norb must be in [1, 128]");
    if (n_elec < 0 || n_elec > norb) return sbd_fail(ctx, SBD_EINVAL, "n_elec must be in [0, norb]");
    if (n < 0 || (n > 0 && !words)) return sbd_fail(ctx, SBD_EINVAL, "bad string array");
    if (n >= (i64)INT32_MAX) return sbd_fail(ctx, SBD_EINVAL, "too many strings for int32 indexing");
    const u64 hi_mask = norb >= 128 ? 0 : norb > 64 ? ~0ull << (norb - 64) : ~0ull;
    const u64 lo_mask = norb >= 64 ? 0 : ~0ull << norb;
    for (i64 i = 0; i < n; ++i) {  // SelectedBasis._validate_strings, basis.py:185-194
        const u64 lo = words[2 * i], hi = words[2 * i + 1];
        char buf[160];
        if ((lo & lo_mask) || (hi & hi_mask)) {
            snprintf(buf, sizeof buf, "string %lld (%#llx:%016llx) has bits above orbital %d", (long long)i,
                     (unsigned long long)hi, (unsigned long long)lo, norb - 1);
            return sbd_fail(ctx, SBD_EINVAL, buf);
        }
        const int pc = __builtin_popcountll(lo) + __builtin_popcountll(hi);
        if (pc != n_elec) {
            snprintf(buf, sizeof buf, "string %lld (%#llx:%016llx) has %d electrons, expected %d", (long long)i,
                     (unsigned long long)hi, (unsigned long long)lo, pc, n_elec);
            return sbd_fail(ctx, SBD_EINVAL, buf);
        }
    }
    s.n = n;
    s.n_elec = n_elec;
    s.present = true;
    ctx->t128_norb = norb;
    SBD_CUDA(ctx, s.str.ensure(2 * sizeof(u64) * (n ? n : 1)));
    if (n) SBD_CUDA(ctx, cudaMemcpyAsync(s.str.p, words, 2 * sizeof(u64) * n, cudaMemcpyHostToDevice, ctx->stream));
    int rc = sbd_sort_strings128(ctx, s, norb);
    if (rc) return rc;
    rc = sbd_build_sector_tables128(ctx, s, norb);
    if (rc) return rc;
    s.built = true;
    return SBD_OK;
}

int sbd_table128_counts(sbd_ctx *ctx, int64_t *n_strings, int64_t *n_singles, int64_t *n_doubles) {
    SBD_CHECK_CTX(ctx);
    const Sector &s = ctx->t128;
    if (!s.built) return sbd_fail(ctx, SBD_EINVAL, "128-bit table not built");
    if (n_strings) *n_strings = s.n;
    if (n_singles) *n_singles = s.ns;
    if (n_doubles) *n_doubles = s.nd;
    return SBD_OK;
}

int sbd_table128_export(sbd_ctx *ctx, int64_t *s_off, int64_t *s_tgt, int16_t *s_hole, int16_t *s_part,
                        int8_t *s_phase, int64_t *d_off, int64_t *d_tgt, int16_t *d_h1, int16_t *d_h2, int16_t *d_p1,
                        int16_t *d_p2, int8_t *d_phase) {
    SBD_CHECK_CTX(ctx);
    Sector &s = ctx->t128;
    if (!s.built) return sbd_fail(ctx, SBD_EINVAL, "128-bit table not built");
    return export_sector(ctx, s, s_off, s_tgt, s_hole, s_part, s_phase, d_off, d_tgt, d_h1, d_h2, d_p1, d_p2, d_phase);
}

int sbd_table128_sorted(sbd_ctx *ctx, uint64_t *sorted_words_host, int64_t *perm_host) {
    SBD_CHECK_CTX(ctx);
    Sector &s = ctx->t128;
    if (!s.built) return sbd_fail(ctx, SBD_EINVAL, "128-bit table not built");
    SBD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    int rc = copy_down(ctx, sorted_words_host, s.sorted, 2 * s.n);
    rc |= copy_down_i32_to_i64(ctx, perm_host, s.perm, s.n);
    return rc ? SBD_ECUDA : SBD_OK;
}

int sbd_set_row_window(sbd_ctx *ctx, int64_t lo, int64_t hi) {
    SBD_CHECK_CTX(ctx);
    if (!ctx->sec[0].present) return sbd_fail(ctx, SBD_EINVAL, "alpha strings not set");
    if (ctx->explicit_mode) return sbd_fail(ctx, SBD_EINVAL, "row windows apply to product-mode bases only");
    if (ctx->dist.on && ctx->dist.nranks > 1)
        return sbd_fail(ctx, SBD_EINVAL, "the row window of a distributed context is its partition block");
    if (!(0 <= lo && lo <= hi && hi <= ctx->sec[0].n))
        return sbd_fail(ctx, SBD_EINVAL, "alpha window (" + std::to_string(lo) + ", " + std::to_string(hi) +
                                             ") exceeds basis");
    ctx->row_lo = lo;
    ctx->row_hi = hi;
    ctx->diag_valid = false;
    return SBD_OK;
}

}  // extern "C"
