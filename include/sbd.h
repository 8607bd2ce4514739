/*
 * sbd.h -- C ABI of the B200-native Selected Basis Diagonalization backend.
 *
 * The reference package (`sbdiag`, arxiv 2601.16637) has no C ABI: its
 * drop-in boundary is the Python operator protocol consumed by
 * `davidson_solve` (pkg/src/sbdiag/davidson.py:191-196,242):
 *
 *     apply_h(x: float64[N]) -> float64[N]   plus   diag: float64[N]
 *
 * implemented by `HamiltonianApplier` (apply.py:651-704) and
 * `DistributedApplier` (distsim.py:130-316).  Every entry point below
 * replaces one piece of that stack; the reference interface it stands in for
 * is cited beside it.  The Python package `paper_2601_16637_b200` binds this
 * header with ctypes and re-exposes the reference API.
 *
 * Conventions
 *   - every call returns SBD_OK (0), SBD_EINVAL (1, -> ValueError) or
 *     SBD_ECUDA (2, -> RuntimeError); sbd_last_error() describes the failure;
 *   - pointers named *_host are host memory, *_dev device memory on the
 *     context's GPU; all device work is ordered on the context's stream
 *     (sbd_set_stream), and calls returning host data synchronise it;
 *   - strings are uint64 occupation masks (bit p = orbital p, norb <= 64) in
 *     CALLER order; determinant (ia, ib) has index ia*n_beta + ib
 *     (basis.py:208-213);
 *   - integrals use the reference layout: h[norb*norb] row-major,
 *     eri[npair*(npair+1)/2] tri-of-tri (integrals.py:39-41,94-97).
 */
#ifndef SBD_B200_H
#define SBD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBD_OK 0
#define SBD_EINVAL 1
#define SBD_ECUDA 2

#define SBD_SPIN_ALPHA 0
#define SBD_SPIN_BETA 1

typedef struct sbd_ctx sbd_ctx;

/* library / error plumbing */
int sbd_abi_version(void);
const char *sbd_last_error(const sbd_ctx *ctx); /* ctx may be NULL: thread-global last error */

/* Context lifetime.  Replaces HamiltonianApplier.__init__ state ownership
 * (apply.py:659-686): the context owns tables, diagonal and scratch. */
int sbd_create(int device, sbd_ctx **out);
int sbd_destroy(sbd_ctx *ctx);
int sbd_set_stream(sbd_ctx *ctx, void *cuda_stream); /* NULL = legacy default stream */

/* IntegralTable upload (integrals.py:44-103). */
int sbd_set_integrals(sbd_ctx *ctx, int norb, const double *h_host, const double *eri_host,
                      int64_t n_eri, double e_core);

/* One spin sector's string list, caller order (SelectedBasis.product,
 * basis.py:138-160).  Validates popcount == n_elec and bits < norb. */
int sbd_set_strings(sbd_ctx *ctx, int spin, const uint64_t *strings_host, int64_t n, int n_elec);

/* Explicit (full-bitstring) determinant list, caller order (SelectedBasis.explicit,
 * basis.py:163-180; HamiltonianApplier explicit branch, apply.py:675-683).  The
 * unique alpha and beta strings become the two sectors (first-seen order);
 * sbd_build_tables then also builds the (alpha, beta)-sorted determinant index
 * (duplicates -> SBD_EINVAL), and sbd_diag / sbd_sigma / sbd_sigma_host act on
 * the n determinants in caller order (_explicit_kernel, apply.py:429-444).  Row
 * windows and the split sigma are product-mode only. */
int sbd_set_dets(sbd_ctx *ctx, const uint64_t *alpha_host, const uint64_t *beta_host, int64_t n,
                 int n_alpha_elec, int n_beta_elec);

/* Device ingestion of sampled determinants (ingest_samples, basis.py:251-313):
 * samples whose per-spin popcount differs from the electron counts are
 * filtered, duplicates dropped keeping FIRST-SEEN order, multiplicities
 * counted (det_counts), and the unique alpha / beta halves collected in
 * first-seen order.  Bits at or above norb -> SBD_EINVAL.  Results stay in the
 * context until sbd_ingest_export copies them out (any pointer may be NULL). */
int sbd_ingest_samples(sbd_ctx *ctx, const uint64_t *alpha_host, const uint64_t *beta_host, int64_t n, int norb,
                       int n_alpha_elec, int n_beta_elec, int64_t *n_filtered, int64_t *n_unique_dets,
                       int64_t *n_unique_alpha, int64_t *n_unique_beta);
int sbd_ingest_export(sbd_ctx *ctx, uint64_t *det_alpha_host, uint64_t *det_beta_host, int64_t *det_count_host,
                      uint64_t *alpha_strings_host, uint64_t *beta_strings_host);

/* Configuration processing + excitation generation on the device:
 * radix sort/unique of each sector's strings, CSR in-set singles/doubles
 * with phases (build_excitation_table, basis.py:362-403; build_spin_tables,
 * apply.py:557-563), per-entry Slater-Condon coefficients and the
 * diagonal building blocks.  Duplicated strings -> SBD_EINVAL. */
int sbd_build_tables(sbd_ctx *ctx);

/* Table sizes and bit-exact export in the reference's column layout
 * (ExcitationTable, basis.py:316-338); any pointer may be NULL to skip. */
int sbd_table_counts(sbd_ctx *ctx, int spin, int64_t *n_strings, int64_t *n_singles, int64_t *n_doubles);
int sbd_export_table(sbd_ctx *ctx, int spin,
                     int64_t *s_off_host, int64_t *s_tgt_host, int16_t *s_hole_host,
                     int16_t *s_part_host, int8_t *s_phase_host,
                     int64_t *d_off_host, int64_t *d_tgt_host, int16_t *d_hole1_host,
                     int16_t *d_hole2_host, int16_t *d_part1_host, int16_t *d_part2_host,
                     int8_t *d_phase_host);
/* Sorted strings and sort permutation (sorted[i] = strings[perm[i]]). */
int sbd_export_sorted(sbd_ctx *ctx, int spin, uint64_t *sorted_host, int64_t *perm_host);

/* 128-bit strings (norb <= 128): configuration processing and excitation
 * generation only.  The reference's table builder works on Python ints of any
 * width (enumerate_singles/doubles, build_excitation_table: basis.py:62-103,
 * 362-403); its integrals stop at 64 orbitals (integrals.py:67-68), so there is
 * no sigma for these strings.  words_host holds n (lo, hi) pairs: string i =
 * words[2i] | words[2i+1] << 64.  Needs no integrals; replaces the table the
 * previous call built.  Bits above norb-1 or a wrong electron count ->
 * SBD_EINVAL (basis.py:185-194); duplicated strings -> SBD_EINVAL. */
int sbd_table128_build(sbd_ctx *ctx, int norb, const uint64_t *words_host, int64_t n, int n_elec);
int sbd_table128_counts(sbd_ctx *ctx, int64_t *n_strings, int64_t *n_singles, int64_t *n_doubles);
int sbd_table128_export(sbd_ctx *ctx,
                        int64_t *s_off_host, int64_t *s_tgt_host, int16_t *s_hole_host,
                        int16_t *s_part_host, int8_t *s_phase_host,
                        int64_t *d_off_host, int64_t *d_tgt_host, int16_t *d_hole1_host,
                        int16_t *d_hole2_host, int16_t *d_part1_host, int16_t *d_part2_host,
                        int8_t *d_phase_host);
/* Sorted (lo, hi) pairs and the sort permutation. */
int sbd_table128_sorted(sbd_ctx *ctx, uint64_t *sorted_words_host, int64_t *perm_host);

/* Rows this context owns: alpha rows [alpha_lo, alpha_hi) x all beta
 * (make_partition semantics, distsim.py:63-77).  Default: all rows. */
int sbd_set_row_window(sbd_ctx *ctx, int64_t alpha_lo, int64_t alpha_hi);

/* Hamiltonian diagonal of the owned rows (compute_diagonal, apply.py:573-586). */
int sbd_diag(sbd_ctx *ctx, double *out_dev);

/* sigma = H x for the owned rows (HamiltonianApplier.__call__, apply.py:688-695;
 * _apply_product, apply.py:608-623).  x_full_dev holds ALL n_alpha*n_beta
 * amplitudes, y_dev the owned rows.  Row-owned, no atomics on y. */
int sbd_sigma(sbd_ctx *ctx, const double *x_full_dev, double *y_dev);

/* nvec sigmas in one call (the block form SURVEY 8(b) lists: Davidson with block expansion, several
 * roots): vector v is x_full_dev + v * ldx, its result y_dev + v * ldy (ldx >= n_alpha*n_beta,
 * ldy >= owned determinants).  Stream-ordered, one vector after the other. */
int sbd_sigma_multi(sbd_ctx *ctx, const double *x_full_dev, int64_t ldx, double *y_dev, int64_t ldy, int nvec);

/* Split form for multi-GPU overlap (the ring of distsim.py:200-259):
 *   sbd_sigma_local  -- beta-beta part from the OWNED rows only (no remote data);
 *   sbd_sigma_remote -- alpha-alpha + alpha-beta part once x_full is gathered,
 *                       combined with the local part into y_dev. */
int sbd_sigma_local(sbd_ctx *ctx, const double *x_own_dev);
int sbd_sigma_remote(sbd_ctx *ctx, const double *x_full_dev, double *y_dev);

/* End-to-end form: host x (all rows) in, host y (owned rows) out; H2D and D2H
 * happen inside the call on the context's stream (numpy protocol of
 * davidson.py:242). */
int sbd_sigma_host(sbd_ctx *ctx, const double *x_full_host, double *y_host);

/* Independent dense check rows (verify's matrix; oracle.assemble_dense, oracle.py:34-45):
 * out[r * N + j] = <det(row0 + r)|H|det(j)> for r < nrows, every element evaluated
 * from the two determinants' words (_hij_words, apply.py:152-177) -- no tables,
 * no sigma kernels.  Needs only sbd_set_integrals + strings (or sbd_set_dets). */
int sbd_dense_rows(sbd_ctx *ctx, int64_t row0, int64_t nrows, double *out_dev);

/* Mean in-set alpha connections per alpha string (c-bar)
 * and the algorithmic sigma bytes 8*N_own*(3 + c-bar). */
int sbd_sigma_model(sbd_ctx *ctx, double *cbar_alpha, double *bytes_per_sigma);
/* Which task-0 kernel (the alpha-single x beta-single term, apply.py:228-238) the last sigma ran:
 * 0 none, 1 SELL cluster multicast, 2 SELL TMA-staged, 3 SELL flat, 4 direct-CI on DMMA. */
int sbd_last_task0(sbd_ctx *ctx, int *kind);

/* ---- Multi-GPU: alpha-block partition, one context (process) per GPU ----
 * Replaces DistributedApplier (distsim.py:130-316) and its ring
 * (distsim.py:200-259) with NCCL over NVLink/NVSwitch, resolved at run time
 * from libnccl.so.2 (the already-loaded one inside PyTorch processes).
 *
 *   sbd_nccl_unique_id  -- rank 0 makes the 128-byte id; the caller broadcasts it
 *                          (ncclGetUniqueId);
 *   sbd_dist_init       -- collective: joins the communicator and takes the
 *                          make_partition block of `rank` (distsim.py:63-77),
 *                          or block `rank` of the caller's alpha_edges, as
 *                          the row window.  Call after sbd_set_strings, before
 *                          (or after) sbd_build_tables.  nranks = 1 needs no id;
 *   sbd_dist_plan       -- collective, optional (sbd_sigma_dist plans with the
 *                          defaults 0, 0.6, 2): exchange 0 auto / 1 dense (whole
 *                          blocks) / 2 sparse (only the referenced rows; auto picks
 *                          sparse when the largest referenced fraction of remote
 *                          rows is <= sparse_threshold); group_steps ring steps
 *                          per pipelined alpha pass;
 *   sbd_sigma_dist      -- collective: y_own = (H x)[own rows] from x_own (this
 *                          rank's rows only), exchange overlapped with the beta
 *                          side and the passes over already-landed blocks;
 *   sbd_dist_allreduce  -- in-place all-reduce of n device doubles (0 sum, 1 max,
 *                          2 min) on the context's stream;
 *   sbd_dist_check      -- NCCL asynchronous error -> SBD_ECUDA;
 *   sbd_dist_info       -- partition and plan (recv/send rows per sigma);
 *   sbd_dist_set_profiling / sbd_dist_stats -- per ring step (0 = local work,
 *                          g = group g) compute / transfer / exposed device
 *                          milliseconds summed over the profiled sigmas
 *                          (StepStat / overlap_stats, distsim.py:81-88,340-367).
 * sbd_davidson on a partitioned context solves over the rank's rows with the
 * dot products all-reduced (every rank calls it; x0 / evecs are local rows). */
int sbd_nccl_unique_id(char *id_out /* 128 bytes */);
int sbd_dist_init(sbd_ctx *ctx, int rank, int nranks, const char *id /* 128 bytes */,
                  const int64_t *alpha_edges /* nranks + 1 block edges, or NULL: make_partition */);
int sbd_dist_plan(sbd_ctx *ctx, int exchange, double sparse_threshold, int group_steps);
int sbd_sigma_dist(sbd_ctx *ctx, const double *x_own_dev, double *y_own_dev);
int sbd_dist_allreduce(sbd_ctx *ctx, double *buf_dev, int64_t n, int op);
int sbd_dist_check(sbd_ctx *ctx);
int sbd_dist_info(sbd_ctx *ctx, int *rank, int *nranks, int64_t *alpha_lo, int64_t *alpha_hi, int *sparse,
                  double *needed_fraction, int64_t *recv_rows, int64_t *send_rows, int *n_groups);
int sbd_dist_set_profiling(sbd_ctx *ctx, int on);
int sbd_dist_stats(sbd_ctx *ctx, int64_t *n_sigma, int *n_steps, double *compute_ms, double *transfer_ms,
                   double *exposed_ms, double *total_ms);

/* ---- Davidson building blocks (davidson.py), all device-resident ---- */

/* out[i] = <V_i, w> for i < k; V_i = V + i*ldv.  Partial per-rank sums
 * (all-reduce them for multi-GPU).  out_dev has k doubles. */
int sbd_vdots(sbd_ctx *ctx, const double *V_dev, int k, int64_t ldv, int64_t n,
              const double *w_dev, double *out_dev);

/* One pass, two right-hand sides: out[i] = <V_i, w>, out[k + i] = <V_i, u>
 * (projected-matrix column davidson.py:248-249 and the Gram row of the
 * newest basis vector used for ortho_history, davidson.py:260-263). */
int sbd_vdots2(sbd_ctx *ctx, const double *V_dev, int k, int64_t ldv, int64_t n, const double *w_dev,
               const double *u_dev, double *out_dev);

/* Fused Ritz/residual/preconditioner (davidson.py:252-258,277-278,159-163):
 * for j < m: r_j = sum_i Y[i,j] W_i - theta_j sum_i Y[i,j] V_i; t_j = precond(r_j)
 * written to T + j*ldt.  Output (k + 1 + m doubles, device):
 *   out[0:k] = <V_i, t_target>, out[k] = |t_target|^2, out[k+1+j] = |r_j|^2.
 * Y is k x m row-major, theta m doubles, both on the device; m <= 8.
 * sbd_residual_precond is the target = 0 form with rn2 == proj + k + 1. */
int sbd_residual_precond(sbd_ctx *ctx, const double *V_dev, const double *W_dev, int k, int64_t ldv,
                         int64_t n, const double *Y_dev, const double *theta_dev, int m,
                         const double *diag_dev, double delta, double *T_dev, int64_t ldt,
                         double *rn2_dev, double *proj_dev);
int sbd_residual_precond_target(sbd_ctx *ctx, const double *V_dev, const double *W_dev, int k, int64_t ldv,
                                int64_t n, const double *Y_dev, const double *theta_dev, int m, int target,
                                const double *diag_dev, double delta, double *T_dev, int64_t ldt,
                                double *out_dev);

/* Block Gram-Schmidt step (CGS pass of orthogonalize, davidson.py:166-185):
 * t <- t - sum_i c[i] V_i, then out2[i] = <V_i, t> (next pass) and
 * out2[k] = |t|^2.  out2_dev has k+1 doubles.  The _nodots form only
 * writes |t|^2 to out2_dev[0] (last pass). */
int sbd_gs_update(sbd_ctx *ctx, const double *V_dev, int k, int64_t ldv, int64_t n,
                  const double *c_dev, double *t_dev, double *out2_dev);
int sbd_gs_update_nodots(sbd_ctx *ctx, const double *V_dev, int k, int64_t ldv, int64_t n,
                         const double *c_dev, double *t_dev, double *out_norm2_dev);

/* Last CGS pass fused with normalisation: v_out = (t - sum_i c[i] V_i) * (*scale_dev),
 * t untouched; out_norm2_dev[0] = |t - V c|^2 (before scaling).  The caller
 * takes scale = 1/sqrt(|t|^2 - |c|^2), exact for orthonormal V.  On the non-TMA
 * fallback path t is overwritten with t - V c. */
int sbd_gs_finalize(sbd_ctx *ctx, const double *V_dev, int k, int64_t ldv, int64_t n, const double *c_dev,
                    const double *t_dev, double *v_out_dev, const double *scale_dev, double *out_norm2_dev);

/* dst = src * (*scale_dev)  (normalisation, scale stays on the device). */
int sbd_scale_copy(sbd_ctx *ctx, const double *src_dev, double *dst_dev, int64_t n, const double *scale_dev);

/* Thick restart (davidson.py:280-289): V[:,0:keep] <- V[:,0:k] . Y[:, 0:keep]
 * in place (Y k x keep row-major on the device). */
int sbd_rotate(sbd_ctx *ctx, double *V_dev, int k, int64_t ldv, int64_t n, const double *Y_dev, int keep);

/* Ritz vectors U_j = sum_i Y[i,j] V_i (davidson.py:256), j < m. */
int sbd_combine(sbd_ctx *ctx, const double *V_dev, int k, int64_t ldv, int64_t n,
                const double *Y_dev, int m, double *U_dev, int64_t ldu);

/* Projected eigensolve on the device (jacobi_eigh, davidson.py:86-148):
 * A k x k (row-major, symmetrised inside) -> ascending evals, evec columns
 * (row-major k x k).  info_dev[0] = sweeps used (>= max_sweeps: failure). */
int sbd_jacobi(sbd_ctx *ctx, const double *A_dev, int k, int lda, double *evals_dev,
               double *evecs_dev, int max_sweeps, int *info_dev);

/* ---- Native Davidson driver (davidson_solve, davidson.py:191-306) ---- */

/* DavidsonOptions (davidson.py:32-53) with the reference defaults
 * (sbd_davidson_default_opts), plus the B200 orthogonality tracking flag. */
typedef struct sbd_davidson_opts {
    int n_roots;             /* 1 */
    double tol_residual;     /* 1e-8 */
    int max_iters;           /* 200 */
    int max_subspace;        /* 32 (<= 64) */
    int restart_keep;        /* 4 */
    double precond_delta;    /* 1e-6 */
    int reorthogonalize;     /* 1 */
    int track_orthogonality; /* 1: ortho_hist[i] = ||G - I||_F from the fused Gram row */
    int selective_reorth;    /* 0 (reference: always two passes).  1: skip the second
                                Gram-Schmidt pass when |t1| >= |t0| / sqrt(2) after the first
                                ("twice is enough"); B200 extension, reported separately */
} sbd_davidson_opts;

/* DavidsonStats (davidson.py:56-68).  The history pointers are optional
 * caller-owned HOST arrays (NULL = not recorded): theta_hist and res_hist hold
 * max_iters x n_roots doubles (row = iteration, NaN past the roots found),
 * ortho_hist, apply_ms_hist (sigma device time) and iter_ms_hist (host wall
 * time per iteration) max_iters doubles, restart_iters max_iters ints. */
typedef struct sbd_davidson_stats {
    int iterations;
    int converged;
    int n_applies;
    int restarts;
    int breakdowns;
    int n_found;          /* roots returned: min(n_roots, final subspace size) */
    double sigma_ms;      /* summed device time of the sigma builds (CUDA events) */
    double *theta_hist;
    double *res_hist;
    double *ortho_hist;
    double *apply_ms_hist;
    double *iter_ms_hist;
    int *restart_iters;
} sbd_davidson_stats;

int sbd_davidson_default_opts(sbd_davidson_opts *opts);

/* Lowest n_roots eigenpairs of the context's Hamiltonian (product or explicit
 * basis; all rows owned, or a partitioned context from sbd_dist_init, where
 * every rank calls it and vectors are the rank's rows).  diag_dev: the preconditioner's diagonal (N doubles) or
 * NULL for the context's own H_ii (sbd_diag).  x0_dev: start vector (N doubles, normalised inside) or
 * NULL for e_argmin(diag) (davidson.py:219-227).  evals_host / res_norms_host:
 * n_roots doubles; evecs_dev: n_roots rows of ldu doubles (may be NULL).
 * Non-convergence is not an error: stats->converged = 0 (davidson.py:271-275).
 * Jacobi non-convergence returns SBD_ECUDA (RuntimeError, davidson.py:144-145).
 * Breakdown recovery draws its random direction on the device, not from
 * numpy's generator (davidson.py:295). */
int sbd_davidson(sbd_ctx *ctx, const sbd_davidson_opts *opts, const double *diag_dev, const double *x0_dev,
                 double *evals_host, double *res_norms_host, double *evecs_dev, int64_t ldu, sbd_davidson_stats *stats);

#ifdef __cplusplus
}
#endif
#endif
