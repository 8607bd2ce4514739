/*
 * c_solve.c -- a pure-C consumer of include/sbd.h (no Python, no torch).
 *
 * Reads one instance (integrals in the reference layout, caller-order strings,
 * a trial vector), builds the device tables, applies H once through the
 * host-buffer entry point and solves for the lowest roots with the native
 * Davidson driver.  tests/test_gpu_cabi.py writes the input with numpy and
 * checks the outputs against the oracle.
 *
 *   gcc -O2 -I include examples/c_solve.c -L paper_2601_16637_b200 -lsbd_b200 \
 *       -Wl,-rpath,$PWD/paper_2601_16637_b200 -lcudart -o c_solve
 *   ./c_solve in.bin out.bin [n_roots]
 *
 * in.bin : i32 norb, n_alpha_elec, n_beta_elec; i64 n_alpha, n_beta, n_eri; f64 e_core;
 *          f64 h[norb*norb]; f64 eri[n_eri]; u64 alpha[n_alpha]; u64 beta[n_beta]; f64 x[N]
 * out.bin: f64 sigma[N]; i32 iterations, converged, n_found; f64 energies[n_roots]; f64 residuals[n_roots]
 */
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "sbd.h"

#define CHECK(call)                                                                 \
    do {                                                                            \
        int rc_ = (call);                                                           \
        if (rc_ != SBD_OK) {                                                        \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, sbd_last_error(ctx)); \
            return 1;                                                               \
        }                                                                           \
    } while (0)

static int rd(FILE *f, void *p, size_t sz, size_t n) { return fread(p, sz, n, f) == n ? 0 : 1; }

int main(int argc, char **argv) {
    if (argc < 3) {
        fprintf(stderr, "usage: %s in.bin out.bin [n_roots]\n", argv[0]);
        return 2;
    }
    FILE *f = fopen(argv[1], "rb");
    if (!f) return 2;
    int32_t hdr[3];
    int64_t dims[3];
    double e_core;
    if (rd(f, hdr, 4, 3) || rd(f, dims, 8, 3) || rd(f, &e_core, 8, 1)) return 2;
    const int norb = hdr[0];
    const int64_t na = dims[0], nb = dims[1], n_eri = dims[2], n = na * nb;
    double *h = malloc(sizeof(double) * norb * norb), *eri = malloc(sizeof(double) * n_eri);
    uint64_t *a = malloc(8 * na), *b = malloc(8 * nb);
    double *x = malloc(8 * n), *y = malloc(8 * n);
    if (rd(f, h, 8, (size_t)norb * norb) || rd(f, eri, 8, n_eri) || rd(f, a, 8, na) || rd(f, b, 8, nb) ||
        rd(f, x, 8, n))
        return 2;
    fclose(f);
    const int n_roots = argc > 3 ? atoi(argv[3]) : 1;

    sbd_ctx *ctx = NULL;
    CHECK(sbd_create(0, &ctx));
    CHECK(sbd_set_integrals(ctx, norb, h, eri, n_eri, e_core));
    CHECK(sbd_set_strings(ctx, SBD_SPIN_ALPHA, a, na, hdr[1]));
    CHECK(sbd_set_strings(ctx, SBD_SPIN_BETA, b, nb, hdr[2]));
    CHECK(sbd_build_tables(ctx));
    CHECK(sbd_sigma_host(ctx, x, y)); /* the numpy protocol of davidson.py:242, from C */

    sbd_davidson_opts opts;
    CHECK(sbd_davidson_default_opts(&opts));
    opts.n_roots = n_roots;
    sbd_davidson_stats st = {0};
    double evals[8], res[8];
    double *evecs = NULL;
    if (cudaMalloc((void **)&evecs, sizeof(double) * n * n_roots) != cudaSuccess) return 3;
    CHECK(sbd_davidson(ctx, &opts, NULL, NULL, evals, res, evecs, n, &st));
    cudaFree(evecs);
    CHECK(sbd_destroy(ctx));

    FILE *o = fopen(argv[2], "wb");
    if (!o) return 2;
    int32_t info[3] = {st.iterations, st.converged, st.n_found};
    fwrite(y, 8, n, o);
    fwrite(info, 4, 3, o);
    fwrite(evals, 8, n_roots, o);
    fwrite(res, 8, n_roots, o);
    fclose(o);
    printf("c_solve: N=%lld E0=%.12f iterations=%d converged=%d\n", (long long)n, evals[0], st.iterations,
           st.converged);
    free(h), free(eri), free(a), free(b), free(x), free(y);
    return 0;
}
