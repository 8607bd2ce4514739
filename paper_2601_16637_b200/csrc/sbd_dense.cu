// Dense Hamiltonian rows from determinant words: the independent check
// matrix of `verify` (reference cli.py:263-272 -> oracle.assemble_dense,
// oracle.py:34-54, which evaluates matelem per element).
//
// One thread per element evaluates <bra|H|ket> from the two determinants'
// occupation words alone, restating _hij_words (apply.py:152-177) with its
// helpers (_hdiag_words, _single_elem, _same_spin_double, apply.py:84-150).
// Nothing here touches the sigma path's machinery -- no excitation tables,
// no per-entry coefficients, no J tables, no sign-folded ERI rows -- so a
// Davidson energy of the sigma operator that matches the eigenvalues of
// this matrix checks the operator independently.
#include "sbd_internal.cuh"

namespace {

__device__ __forceinline__ int ctz64(u64 w) { return __ffsll((long long)w) - 1; }
__device__ __forceinline__ u64 bit64(int p) { return (u64)1 << p; }

// (-1)^(occupied bits of w strictly between p and r)  (_single_sign, apply.py:67-73)
__device__ __forceinline__ double single_sign(u64 w, int p, int r) {
    const int lo = p < r ? p : r, hi = p < r ? r : p;
    const u64 mask = (bit64(hi) - 1) & ~(bit64(lo + 1) - 1);
    return (__popcll(w & mask) & 1) ? -1.0 : 1.0;
}

__device__ __forceinline__ double eri4(const double *__restrict__ eri, int p, int q, int r, int s) {
    const i64 a = tri_idx(p, q), b = tri_idx(r, s);
    return __ldg(eri + tri_idx(a, b));
}

__device__ double sector_diag(u64 w0, const double *__restrict__ h, int norb, const double *__restrict__ eri) {
    double e = 0.0;
    for (u64 t = w0; t; t &= t - 1) {
        const int p = ctz64(t);
        e += __ldg(h + p * norb + p);
        for (u64 t2 = w0; t2; t2 &= t2 - 1) {
            const int q = ctz64(t2);
            e += 0.5 * (eri4(eri, p, p, q, q) - eri4(eri, p, q, q, p));
        }
    }
    return e;
}

__device__ double single_elem(u64 mb, u64 mk, u64 other, const double *__restrict__ h, int norb,
                              const double *__restrict__ eri) {
    const u64 x = mb ^ mk;
    const int p = ctz64(x & mb), r = ctz64(x & mk);
    double elem = __ldg(h + p * norb + r);
    for (u64 t = mb & mk; t; t &= t - 1) {
        const int q = ctz64(t);
        elem += eri4(eri, p, r, q, q) - eri4(eri, p, q, q, r);
    }
    for (u64 t = other; t; t &= t - 1) elem += eri4(eri, p, r, ctz64(t), ctz64(t));
    return single_sign(mb, p, r) * elem;
}

__device__ double same_spin_double(u64 wb, u64 wk, const double *__restrict__ eri) {
    const u64 x = wb ^ wk, holes = x & wb, parts = x & wk;
    const int p = ctz64(holes), q = ctz64(holes & (holes - 1));
    const int r = ctz64(parts), s = ctz64(parts & (parts - 1));
    double sign = single_sign(wb, p, r);
    const u64 inter = (wb & ~bit64(p)) | bit64(r);
    sign *= single_sign(inter, q, s);
    return sign * (eri4(eri, p, r, q, s) - eri4(eri, p, s, q, r));
}

__device__ double hij_words(u64 ba, u64 bb, u64 ka, u64 kb, const double *__restrict__ h, int norb,
                            const double *__restrict__ eri, double e_core) {
    const u64 xa = ba ^ ka, xb = bb ^ kb;
    const int na = __popcll(xa), nb = __popcll(xb), d2 = na + nb;
    if (d2 == 0) {
        double e = e_core + sector_diag(ba, h, norb, eri) + sector_diag(bb, h, norb, eri);
        for (u64 ta = ba; ta; ta &= ta - 1)
            for (u64 tb = bb; tb; tb &= tb - 1) e += eri4(eri, ctz64(ta), ctz64(ta), ctz64(tb), ctz64(tb));
        return e;
    }
    if (d2 == 2) return na == 2 ? single_elem(ba, ka, bb, h, norb, eri) : single_elem(bb, kb, ba, h, norb, eri);
    if (d2 == 4) {
        if (na == 2) {  // opposite-spin double
            const int pa = ctz64(xa & ba), ra = ctz64(xa & ka), pb = ctz64(xb & bb), rb = ctz64(xb & kb);
            return single_sign(ba, pa, ra) * single_sign(bb, pb, rb) * eri4(eri, pa, ra, pb, rb);
        }
        return na == 4 ? same_spin_double(ba, ka, eri) : same_spin_double(bb, kb, eri);
    }
    return 0.0;
}

// determinant words of index i: product (ia * nb + ib) or explicit (caller-order list)
struct Dets {
    const u64 *astr, *bstr;
    const int32_t *da, *db;  // explicit only
    i64 nb;
    __device__ __forceinline__ void words(i64 i, u64 &a, u64 &b) const {
        if (da) {
            a = astr[da[i]];
            b = bstr[db[i]];
        } else {
            a = astr[i / nb];
            b = bstr[i % nb];
        }
    }
};

__global__ void dense_rows_kernel(Dets d, i64 row0, i64 nrows, i64 n, const double *__restrict__ h, int norb,
                                  const double *__restrict__ eri, double e_core, double *__restrict__ out) {
    const i64 total = nrows * n;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (i64)gridDim.x * blockDim.x) {
        const i64 r = e / n, j = e - r * n;
        u64 ba, bb, ka, kb;
        d.words(row0 + r, ba, bb);
        d.words(j, ka, kb);
        out[e] = hij_words(ba, bb, ka, kb, h, norb, eri, e_core);
    }
}

}  // namespace

extern "C" {

int sbd_dense_rows(sbd_ctx *ctx, int64_t row0, int64_t nrows, double *out_dev) {
    SBD_CHECK_CTX(ctx);
    if (!ctx->have_integrals || !ctx->sec[0].present || !ctx->sec[1].present)
        return sbd_fail(ctx, SBD_EINVAL, "integrals and strings must be set first");
    Dets d{ctx->sec[0].str.as<u64>(), ctx->sec[1].str.as<u64>(), nullptr, nullptr, ctx->sec[1].n};
    i64 n = ctx->sec[0].n * ctx->sec[1].n;
    if (ctx->explicit_mode) {
        d.da = ctx->det_a.as<int32_t>();
        d.db = ctx->det_b.as<int32_t>();
        n = ctx->n_det;
    }
    if (row0 < 0 || nrows < 0 || row0 + nrows > n) return sbd_fail(ctx, SBD_EINVAL, "dense rows out of range");
    if (nrows == 0 || n == 0) return SBD_OK;
    if (!out_dev) return sbd_fail(ctx, SBD_EINVAL, "null output");
    const unsigned blocks = (unsigned)std::min<i64>(grid_for(nrows * n, 256), 16 * (i64)ctx->num_sms);
    dense_rows_kernel<<<blocks, 256, 0, ctx->stream>>>(d, row0, nrows, n, ctx->h.as<double>(), ctx->norb,
                                                        ctx->eri.as<double>(), ctx->e_core, out_dev);
    SBD_LAUNCHED(ctx, "dense_rows_kernel");
    return SBD_OK;
}

}  // extern "C"
