/*
 * sbd_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU algorithm for the SBD hot
 * path (arxiv 2601.16637 reference package `sbdiag`, numba kernels in
 * pkg/src/sbdiag/apply.py and the pure-Python table builder in basis.py).
 * It is the checker for the CUDA path and the CPU baseline arm of bench.py
 * (cpu_baseline.kind = "port").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the product
 * package never does.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every entry point
 * against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py, run with /root/reference importable).
 *
 * Floating point follows the reference's operation order; build with
 * -ffp-contract=off so no FMA contraction changes rounding.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>
#include <unistd.h>

typedef uint64_t u64;
typedef int64_t i64;

static inline int popc(u64 w) { return __builtin_popcountll(w); }
static inline int ctz(u64 w) { return __builtin_ctzll(w); }
static inline u64 bit(int p) { return (u64)1 << p; }

/* apply.py:68-74 / basis.py:62-69: (-1)^(occupied bits strictly between p and r) */
static inline double sign_between(u64 w, int p, int r) {
    int lo = p < r ? p : r, hi = p < r ? r : p;
    u64 mask = (bit(hi) - 1) & ~(bit(lo + 1) - 1);
    return (popc(w & mask) & 1) ? -1.0 : 1.0;
}
static inline int iphase_between(u64 w, int p, int r) { return sign_between(w, p, r) < 0 ? -1 : 1; }

/* apply.py:77-81: 8-fold folded ERI gather */
static inline i64 tri(i64 a, i64 b) { return a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a; }
static inline double eri_at(const double *eri, int p, int q, int r, int s) {
    return eri[tri(tri(p, q), tri(r, s))];
}

/* apply.py:84-97 */
static double sector_diag(u64 w0, const double *h, int norb, const double *eri) {
    double e = 0.0;
    for (u64 t = w0; t; t &= t - 1) {
        int p = ctz(t);
        e += h[p * norb + p];
        for (u64 t2 = w0; t2; t2 &= t2 - 1) {
            int q = ctz(t2);
            e += 0.5 * (eri_at(eri, p, p, q, q) - eri_at(eri, p, q, q, p));
        }
    }
    return e;
}

/* apply.py:100-112 */
double orc_hdiag(u64 aw, u64 bw, const double *h, int norb, const double *eri, double e_core) {
    double e = e_core + sector_diag(aw, h, norb, eri) + sector_diag(bw, h, norb, eri);
    for (u64 ta = aw; ta; ta &= ta - 1) {
        int p = ctz(ta);
        for (u64 tb = bw; tb; tb &= tb - 1) e += eri_at(eri, p, p, ctz(tb), ctz(tb));
    }
    return e;
}

/* apply.py:115-134: same-spin single, mb/mk moving sector bra/ket, other = spectator */
static double single_elem(u64 mb, u64 mk, u64 other, const double *h, int norb, const double *eri) {
    u64 x = mb ^ mk;
    int p = ctz(x & mb), r = ctz(x & mk);
    double elem = h[p * norb + r];
    for (u64 t = mb & mk; t; t &= t - 1) {
        int q = ctz(t);
        elem += eri_at(eri, p, r, q, q) - eri_at(eri, p, q, q, r);
    }
    for (u64 t = other; t; t &= t - 1) {
        int q = ctz(t);
        elem += eri_at(eri, p, r, q, q);
    }
    return sign_between(mb, p, r) * elem;
}

/* apply.py:137-149 */
static double same_spin_double(u64 wb, u64 wk, const double *eri) {
    u64 x = wb ^ wk, holes = x & wb, parts = x & wk;
    int p = ctz(holes), q = ctz(holes & (holes - 1));
    int r = ctz(parts), s = ctz(parts & (parts - 1));
    double sgn = sign_between(wb, p, r);
    u64 inter = (wb & ~bit(p)) | bit(r);
    sgn *= sign_between(inter, q, s);
    return sgn * (eri_at(eri, p, r, q, s) - eri_at(eri, p, s, q, r));
}

/* apply.py:152-177: degree dispatch */
double orc_hij(u64 ba, u64 bb, u64 ka, u64 kb, const double *h, int norb, const double *eri, double e_core) {
    u64 xa = ba ^ ka, xb = bb ^ kb;
    int na = popc(xa), nb = popc(xb), d2 = na + nb;
    if (d2 == 0) return orc_hdiag(ba, bb, h, norb, eri, e_core);
    if (d2 == 2) return na == 2 ? single_elem(ba, ka, bb, h, norb, eri) : single_elem(bb, kb, ba, h, norb, eri);
    if (d2 == 4) {
        if (na == 2) {
            int pa = ctz(xa & ba), ra = ctz(xa & ka), pb = ctz(xb & bb), rb = ctz(xb & kb);
            double sgn = sign_between(ba, pa, ra) * sign_between(bb, pb, rb);
            return sgn * eri_at(eri, pa, ra, pb, rb);
        }
        return na == 4 ? same_spin_double(ba, ka, eri) : same_spin_double(bb, kb, eri);
    }
    return 0.0;
}

/* apply.py:183-245: one sigma row, same accumulation order as the reference.
 * x is indexed by the ket window: x[(ja - kalo) * nbeta + jb].            */
static double product_row(i64 bi, const double *x, const double *diag, const u64 *alpha, const u64 *beta,
                          i64 balo, i64 kalo, i64 kahi, i64 nbeta,
                          const i64 *as_off, const i64 *as_tgt, const i64 *ad_off, const i64 *ad_tgt,
                          const i64 *bs_off, const i64 *bs_tgt, const i64 *bd_off, const i64 *bd_tgt,
                          const double *h, int norb, const double *eri, double e_core) {
    i64 ia = balo + bi / nbeta, ib = bi % nbeta;
    u64 da = alpha[ia], db = beta[ib];
    double acc = 0.0;
    if (kalo <= ia && ia < kahi) {
        i64 xoff = (ia - kalo) * nbeta;
        acc += diag[bi] * x[xoff + ib];
        for (i64 k = bs_off[ib]; k < bs_off[ib + 1]; ++k) {
            i64 jb = bs_tgt[k];
            acc += orc_hij(da, db, da, beta[jb], h, norb, eri, e_core) * x[xoff + jb];
        }
        for (i64 k = bd_off[ib]; k < bd_off[ib + 1]; ++k) {
            i64 jb = bd_tgt[k];
            acc += orc_hij(da, db, da, beta[jb], h, norb, eri, e_core) * x[xoff + jb];
        }
    }
    for (i64 k = as_off[ia]; k < as_off[ia + 1]; ++k) {
        i64 ja = as_tgt[k];
        if (kalo <= ja && ja < kahi) {
            i64 joff = (ja - kalo) * nbeta;
            u64 ka = alpha[ja];
            acc += orc_hij(da, db, ka, db, h, norb, eri, e_core) * x[joff + ib];
            for (i64 m = bs_off[ib]; m < bs_off[ib + 1]; ++m) {
                i64 jb = bs_tgt[m];
                acc += orc_hij(da, db, ka, beta[jb], h, norb, eri, e_core) * x[joff + jb];
            }
        }
    }
    for (i64 k = ad_off[ia]; k < ad_off[ia + 1]; ++k) {
        i64 ja = ad_tgt[k];
        if (kalo <= ja && ja < kahi)
            acc += orc_hij(da, db, alpha[ja], db, h, norb, eri, e_core) * x[(ja - kalo) * nbeta + ib];
    }
    return acc;
}

/* Minimal dynamic parallel-for over [0, n) in chunks (the reference uses
 * numba prange with the workqueue layer; rows are independent). */
typedef void (*range_fn)(i64 lo, i64 hi, void *ctx);
typedef struct { i64 n, chunk; i64 next; pthread_mutex_t mu; range_fn fn; void *ctx; } par_job;

static void *par_worker(void *arg) {
    par_job *j = (par_job *)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        i64 lo = j->next;
        j->next += j->chunk;
        pthread_mutex_unlock(&j->mu);
        if (lo >= j->n) break;
        i64 hi = lo + j->chunk < j->n ? lo + j->chunk : j->n;
        j->fn(lo, hi, j->ctx);
    }
    return 0;
}

int orc_max_threads(void) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

static void par_for(i64 n, i64 chunk, int nthreads, range_fn fn, void *ctx) {
    if (nthreads <= 0) nthreads = orc_max_threads();
    if (nthreads > 256) nthreads = 256;
    par_job j = {n, chunk, 0, PTHREAD_MUTEX_INITIALIZER, fn, ctx};
    if (nthreads == 1 || n <= chunk) { fn(0, n, ctx); return; }
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], 0, par_worker, &j);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], 0);
}

/* apply.py:248-311 (_product_kernel_seq/_par): y[bi] += row(bi) for bra rows
 * [balo, bahi) x all beta; rows are independent (prange in the reference). */
typedef struct {
    i64 balo, kalo, kahi, nbeta;
    double *y; const double *x, *diag; const u64 *alpha, *beta;
    const i64 *as_off, *as_tgt, *ad_off, *ad_tgt, *bs_off, *bs_tgt, *bd_off, *bd_tgt;
    const double *h, *eri; int norb; double e_core;
} sigma_job;

static void sigma_range(i64 lo, i64 hi, void *vp) {
    sigma_job *j = (sigma_job *)vp;
    for (i64 bi = lo; bi < hi; ++bi)
        j->y[bi] += product_row(bi, j->x, j->diag, j->alpha, j->beta, j->balo, j->kalo, j->kahi, j->nbeta,
                                j->as_off, j->as_tgt, j->ad_off, j->ad_tgt, j->bs_off, j->bs_tgt,
                                j->bd_off, j->bd_tgt, j->h, j->norb, j->eri, j->e_core);
}

void orc_sigma(i64 balo, i64 bahi, i64 kalo, i64 kahi, i64 nbeta, double *y, const double *x,
               const double *diag, const u64 *alpha, const u64 *beta,
               const i64 *as_off, const i64 *as_tgt, const i64 *ad_off, const i64 *ad_tgt,
               const i64 *bs_off, const i64 *bs_tgt, const i64 *bd_off, const i64 *bd_tgt,
               const double *h, int norb, const double *eri, double e_core, int nthreads) {
    sigma_job j = {balo, kalo, kahi, nbeta, y, x, diag, alpha, beta, as_off, as_tgt, ad_off, ad_tgt,
                   bs_off, bs_tgt, bd_off, bd_tgt, h, eri, norb, e_core};
    par_for((bahi - balo) * nbeta, 256, nthreads, sigma_range, &j);
}

typedef struct { i64 balo, nbeta; double *out; const u64 *alpha, *beta; const double *h, *eri; int norb; double e_core; } diag_job;

static void diag_range(i64 lo, i64 hi, void *vp) {
    diag_job *j = (diag_job *)vp;
    for (i64 i = lo; i < hi; ++i)
        j->out[i] = orc_hdiag(j->alpha[j->balo + i / j->nbeta], j->beta[i % j->nbeta], j->h, j->norb, j->eri, j->e_core);
}

/* apply.py:314-317 + 573-586: diagonal over bra rows [balo, bahi) x beta */
void orc_diag(i64 balo, i64 bahi, i64 nbeta, double *out, const u64 *alpha, const u64 *beta,
              const double *h, int norb, const double *eri, double e_core, int nthreads) {
    diag_job j = {balo, nbeta, out, alpha, beta, h, eri, norb, e_core};
    par_for((bahi - balo) * nbeta, 4096, nthreads, diag_range, &j);
}

/* ---- explicit (full-bitstring) bases: apply.py:320-458 ---- */

/* apply.py:323-335: lower bound on (alpha, beta) over the lexicographically sorted dets */
static i64 find_det(const u64 *sa, const u64 *sb, i64 n, u64 ta, u64 tb) {
    i64 lo = 0, hi = n;
    while (lo < hi) {
        i64 mid = (lo + hi) >> 1;
        u64 a = sa[mid];
        if (a < ta || (a == ta && sb[mid] < tb)) lo = mid + 1;
        else hi = mid;
    }
    if (lo < n && sa[lo] == ta && sb[lo] == tb) return lo;
    return -1;
}

/* apply.py:338-426: one explicit row, the reference's loop nesting and accumulation order */
static double explicit_row(i64 i, const double *x, const double *diag, const u64 *det_a, const u64 *det_b,
                           const u64 *sa, const u64 *sb, const i64 *perm, i64 n, u64 mask, const double *h,
                           int norb, const double *eri, double e_core) {
    const u64 da = det_a[i], db = det_b[i];
    double acc = diag[i] * x[i];
    const u64 va = ~da & mask, vb = ~db & mask;
    for (u64 tp = da; tp; tp &= tp - 1) {  /* alpha singles + their beta-single crosses */
        int p = ctz(tp);
        for (u64 tr = va; tr; tr &= tr - 1) {
            int r = ctz(tr);
            u64 ta = (da & ~bit(p)) | bit(r);
            i64 pos = find_det(sa, sb, n, ta, db);
            if (pos >= 0) acc += orc_hij(da, db, ta, db, h, norb, eri, e_core) * x[perm[pos]];
            for (u64 uq = db; uq; uq &= uq - 1) {
                int q = ctz(uq);
                for (u64 us = vb; us; us &= us - 1) {
                    int s2 = ctz(us);
                    u64 tb = (db & ~bit(q)) | bit(s2);
                    i64 pos2 = find_det(sa, sb, n, ta, tb);
                    if (pos2 >= 0) acc += orc_hij(da, db, ta, tb, h, norb, eri, e_core) * x[perm[pos2]];
                }
            }
        }
    }
    for (u64 tp = db; tp; tp &= tp - 1) {  /* beta singles */
        int q = ctz(tp);
        for (u64 tr = vb; tr; tr &= tr - 1) {
            int s2 = ctz(tr);
            u64 tb = (db & ~bit(q)) | bit(s2);
            i64 pos = find_det(sa, sb, n, da, tb);
            if (pos >= 0) acc += orc_hij(da, db, da, tb, h, norb, eri, e_core) * x[perm[pos]];
        }
    }
    for (int spin = 0; spin < 2; ++spin) {  /* alpha doubles, then beta doubles */
        const u64 w = spin ? db : da, v = spin ? vb : va;
        for (u64 t1 = w; t1; t1 &= t1 - 1) {
            int p = ctz(t1);
            for (u64 t2 = t1 & (t1 - 1); t2; t2 &= t2 - 1) {
                int q = ctz(t2);
                for (u64 u1 = v; u1; u1 &= u1 - 1) {
                    int r = ctz(u1);
                    for (u64 u2 = u1 & (u1 - 1); u2; u2 &= u2 - 1) {
                        int s2 = ctz(u2);
                        u64 t = (w & ~bit(p) & ~bit(q)) | bit(r) | bit(s2);
                        u64 ka = spin ? da : t, kb = spin ? t : db;
                        i64 pos = find_det(sa, sb, n, ka, kb);
                        if (pos >= 0) acc += orc_hij(da, db, ka, kb, h, norb, eri, e_core) * x[perm[pos]];
                    }
                }
            }
        }
    }
    return acc;
}

typedef struct {
    i64 n, i0; double *y; const double *x, *diag; const u64 *det_a, *det_b, *sa, *sb; const i64 *perm;
    u64 mask; const double *h, *eri; int norb; double e_core;
} explicit_job;

static void explicit_range(i64 lo, i64 hi, void *vp) {
    explicit_job *j = (explicit_job *)vp;
    for (i64 i = lo; i < hi; ++i)
        j->y[i] += explicit_row(j->i0 + i, j->x, j->diag, j->det_a, j->det_b, j->sa, j->sb, j->perm, j->n, j->mask,
                                j->h, j->norb, j->eri, j->e_core);
}

/* apply.py:429-444 + 698-703: y = H x over an explicit determinant list (sa/sb/perm from
 * np.lexsort); rows [i0, i1) only (y has i1 - i0 entries, diag is indexed globally) */
void orc_sigma_explicit(i64 n, i64 i0, i64 i1, double *y, const double *x, const double *diag, const u64 *det_a,
                        const u64 *det_b, const u64 *sa, const u64 *sb, const i64 *perm, const double *h, int norb,
                        const double *eri, double e_core, int nthreads) {
    explicit_job j = {n, i0, y, x, diag, det_a, det_b, sa, sb, perm,
                      norb >= 64 ? ~(u64)0 : (bit(norb) - 1), h, eri, norb, e_core};
    par_for(i1 - i0, 64, nthreads, explicit_range, &j);
}

/* ---- excitation tables: basis.py:72-103 (enumeration order) + 362-403 ---- */

typedef struct { u64 key; i64 idx; } keyidx;
static int cmp_keyidx(const void *a, const void *b) {
    u64 x = ((const keyidx *)a)->key, y = ((const keyidx *)b)->key;
    return x < y ? -1 : x > y;
}
/* dict lookup `index.get(target)` restated as binary search over sorted keys */
static i64 lookup(const keyidx *sorted, i64 n, u64 key) {
    i64 lo = 0, hi = n;
    while (lo < hi) {
        i64 mid = (lo + hi) >> 1;
        if (sorted[mid].key < key) lo = mid + 1; else hi = mid;
    }
    return (lo < n && sorted[lo].key == key) ? sorted[lo].idx : -1;
}

/* Enumerate excitations of s; when out arrays are NULL only count.  Returns
 * number of in-set singles in *ns and doubles in *nd. */
static void enum_string(u64 s, int norb, const keyidx *sorted, i64 n, i64 *ns, i64 *nd,
                        i64 *s_tgt, int16_t *s_hole, int16_t *s_part, int8_t *s_phase,
                        i64 *d_tgt, int16_t *d_h1, int16_t *d_h2, int16_t *d_p1, int16_t *d_p2, int8_t *d_phase) {
    int occ[64], virt[64], no = 0, nv = 0;
    for (int o = 0; o < norb; ++o) { if (s >> o & 1) occ[no++] = o; else virt[nv++] = o; }
    i64 cs = 0, cd = 0;
    for (int a = 0; a < no; ++a)               /* basis.py:77-80: p occ asc, r virt asc */
        for (int b = 0; b < nv; ++b) {
            int p = occ[a], r = virt[b];
            u64 t = (s & ~bit(p)) | bit(r);
            i64 j = lookup(sorted, n, t);
            if (j < 0) continue;
            if (s_tgt) { s_tgt[cs] = j; s_hole[cs] = p; s_part[cs] = r; s_phase[cs] = iphase_between(s, p, r); }
            ++cs;
        }
    for (int a = 0; a < no; ++a)               /* basis.py:96-102: combinations(occ,2) x combinations(virt,2) */
        for (int a2 = a + 1; a2 < no; ++a2)
            for (int b = 0; b < nv; ++b)
                for (int b2 = b + 1; b2 < nv; ++b2) {
                    int p = occ[a], q = occ[a2], r = virt[b], so = virt[b2];
                    u64 inter = (s & ~bit(p)) | bit(r);
                    u64 t = (inter & ~bit(q)) | bit(so);
                    i64 j = lookup(sorted, n, t);
                    if (j < 0) continue;
                    if (d_tgt) {
                        d_tgt[cd] = j; d_h1[cd] = p; d_h2[cd] = q; d_p1[cd] = r; d_p2[cd] = so;
                        d_phase[cd] = iphase_between(s, p, r) * iphase_between(inter, q, so);
                    }
                    ++cd;
                }
    *ns = cs; *nd = cd;
}

static keyidx *make_sorted(const u64 *strings, i64 n) {
    keyidx *k = (keyidx *)malloc(sizeof(keyidx) * (n ? n : 1));
    for (i64 i = 0; i < n; ++i) { k[i].key = strings[i]; k[i].idx = i; }
    qsort(k, n, sizeof(keyidx), cmp_keyidx);
    return k;
}

typedef struct {
    const u64 *strings; i64 n; int norb; const keyidx *sorted;
    i64 *s_off, *d_off;
    i64 *s_tgt; int16_t *s_hole, *s_part; int8_t *s_phase;
    i64 *d_tgt; int16_t *d_h1, *d_h2, *d_p1, *d_p2; int8_t *d_phase;
} table_job;

static void count_range(i64 lo, i64 hi, void *vp) {
    table_job *j = (table_job *)vp;
    for (i64 i = lo; i < hi; ++i) {
        i64 ns, nd;
        enum_string(j->strings[i], j->norb, j->sorted, j->n, &ns, &nd, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0);
        j->s_off[i + 1] = ns; j->d_off[i + 1] = nd;
    }
}

static void fill_range(i64 lo, i64 hi, void *vp) {
    table_job *j = (table_job *)vp;
    for (i64 i = lo; i < hi; ++i) {
        i64 ns, nd, so = j->s_off[i], dof = j->d_off[i];
        enum_string(j->strings[i], j->norb, j->sorted, j->n, &ns, &nd, j->s_tgt + so, j->s_hole + so,
                    j->s_part + so, j->s_phase + so, j->d_tgt + dof, j->d_h1 + dof, j->d_h2 + dof,
                    j->d_p1 + dof, j->d_p2 + dof, j->d_phase + dof);
    }
}

/* pass 1: s_off, d_off (len n+1).  Returns -1 if strings are not unique
 * (basis.py:364-366 raises ValueError). */
int orc_table_count(const u64 *strings, i64 n, int norb, i64 *s_off, i64 *d_off, int nthreads) {
    keyidx *sorted = make_sorted(strings, n);
    for (i64 i = 1; i < n; ++i)
        if (sorted[i].key == sorted[i - 1].key) { free(sorted); return -1; }
    s_off[0] = d_off[0] = 0;
    table_job j = {strings, n, norb, sorted, s_off, d_off};
    par_for(n, 16, nthreads, count_range, &j);
    for (i64 i = 0; i < n; ++i) { s_off[i + 1] += s_off[i]; d_off[i + 1] += d_off[i]; }
    free(sorted);
    return 0;
}

/* pass 2: fill the CSR columns given the offsets from pass 1. */
void orc_table_fill(const u64 *strings, i64 n, int norb, const i64 *s_off, const i64 *d_off,
                    i64 *s_tgt, int16_t *s_hole, int16_t *s_part, int8_t *s_phase,
                    i64 *d_tgt, int16_t *d_h1, int16_t *d_h2, int16_t *d_p1, int16_t *d_p2, int8_t *d_phase,
                    int nthreads) {
    keyidx *sorted = make_sorted(strings, n);
    table_job j = {strings, n, norb, sorted, (i64 *)s_off, (i64 *)d_off, s_tgt, s_hole, s_part, s_phase,
                   d_tgt, d_h1, d_h2, d_p1, d_p2, d_phase};
    par_for(n, 16, nthreads, fill_range, &j);
    free(sorted);
}

/* ---- the same tables for strings of up to 128 orbitals (two 64-bit words) ----
 * basis.py:62-103 and 362-403 operate on Python ints of any width; only the integrals are
 * capped at 64 orbitals (integrals.py:67-68).  Strings arrive as (lo, hi) word pairs. */

typedef unsigned __int128 u128;
typedef struct { u128 key; i64 idx; } keyidx128;
static inline u128 bit128(int p) { return (u128)1 << p; }
static inline u128 word128(const u64 *w, i64 i) { return (u128)w[2 * i] | ((u128)w[2 * i + 1] << 64); }
static inline int popc128(u128 w) { return popc((u64)w) + popc((u64)(w >> 64)); }
/* basis.py:62-69 */
static inline int iphase128(u128 w, int p, int r) {
    int lo = p < r ? p : r, hi = p < r ? r : p;
    u128 mask = (bit128(hi) - 1) & ~((bit128(lo) << 1) - 1);
    return popc128(w & mask) & 1 ? -1 : 1;
}
static int cmp_keyidx128(const void *a, const void *b) {
    u128 x = ((const keyidx128 *)a)->key, y = ((const keyidx128 *)b)->key;
    return x < y ? -1 : x > y;
}
static i64 lookup128(const keyidx128 *sorted, i64 n, u128 key) {
    i64 lo = 0, hi = n;
    while (lo < hi) {
        i64 mid = (lo + hi) >> 1;
        if (sorted[mid].key < key) lo = mid + 1; else hi = mid;
    }
    return (lo < n && sorted[lo].key == key) ? sorted[lo].idx : -1;
}

/* basis.py:72-103, same loop nesting as enum_string above */
static void enum_string128(u128 s, int norb, const keyidx128 *sorted, i64 n, i64 *ns, i64 *nd,
                           i64 *s_tgt, int16_t *s_hole, int16_t *s_part, int8_t *s_phase,
                           i64 *d_tgt, int16_t *d_h1, int16_t *d_h2, int16_t *d_p1, int16_t *d_p2, int8_t *d_phase) {
    int occ[128], virt[128], no = 0, nv = 0;
    for (int o = 0; o < norb; ++o) { if ((s >> o) & 1) occ[no++] = o; else virt[nv++] = o; }
    i64 cs = 0, cd = 0;
    for (int a = 0; a < no; ++a)
        for (int b = 0; b < nv; ++b) {
            int p = occ[a], r = virt[b];
            i64 j = lookup128(sorted, n, (s & ~bit128(p)) | bit128(r));
            if (j < 0) continue;
            if (s_tgt) { s_tgt[cs] = j; s_hole[cs] = p; s_part[cs] = r; s_phase[cs] = iphase128(s, p, r); }
            ++cs;
        }
    for (int a = 0; a < no; ++a)
        for (int a2 = a + 1; a2 < no; ++a2)
            for (int b = 0; b < nv; ++b)
                for (int b2 = b + 1; b2 < nv; ++b2) {
                    int p = occ[a], q = occ[a2], r = virt[b], so = virt[b2];
                    u128 inter = (s & ~bit128(p)) | bit128(r);
                    i64 j = lookup128(sorted, n, (inter & ~bit128(q)) | bit128(so));
                    if (j < 0) continue;
                    if (d_tgt) {
                        d_tgt[cd] = j; d_h1[cd] = p; d_h2[cd] = q; d_p1[cd] = r; d_p2[cd] = so;
                        d_phase[cd] = iphase128(s, p, r) * iphase128(inter, q, so);
                    }
                    ++cd;
                }
    *ns = cs; *nd = cd;
}

typedef struct {
    const u64 *words; i64 n; int norb; const keyidx128 *sorted;
    i64 *s_off, *d_off;
    i64 *s_tgt; int16_t *s_hole, *s_part; int8_t *s_phase;
    i64 *d_tgt; int16_t *d_h1, *d_h2, *d_p1, *d_p2; int8_t *d_phase;
} table128_job;

static void count128_range(i64 lo, i64 hi, void *vp) {
    table128_job *j = (table128_job *)vp;
    for (i64 i = lo; i < hi; ++i) {
        i64 ns, nd;
        enum_string128(word128(j->words, i), j->norb, j->sorted, j->n, &ns, &nd, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0);
        j->s_off[i + 1] = ns; j->d_off[i + 1] = nd;
    }
}

static void fill128_range(i64 lo, i64 hi, void *vp) {
    table128_job *j = (table128_job *)vp;
    for (i64 i = lo; i < hi; ++i) {
        i64 ns, nd, so = j->s_off[i], dof = j->d_off[i];
        enum_string128(word128(j->words, i), j->norb, j->sorted, j->n, &ns, &nd, j->s_tgt + so, j->s_hole + so,
                       j->s_part + so, j->s_phase + so, j->d_tgt + dof, j->d_h1 + dof, j->d_h2 + dof,
                       j->d_p1 + dof, j->d_p2 + dof, j->d_phase + dof);
    }
}

static keyidx128 *make_sorted128(const u64 *words, i64 n) {
    keyidx128 *k = (keyidx128 *)malloc(sizeof(keyidx128) * (n ? n : 1));
    for (i64 i = 0; i < n; ++i) { k[i].key = word128(words, i); k[i].idx = i; }
    qsort(k, n, sizeof(keyidx128), cmp_keyidx128);
    return k;
}

/* words: 2n u64, string i = words[2i] | words[2i+1] << 64.  -1 on duplicates (basis.py:364-366). */
int orc_table128_count(const u64 *words, i64 n, int norb, i64 *s_off, i64 *d_off, int nthreads) {
    keyidx128 *sorted = make_sorted128(words, n);
    for (i64 i = 1; i < n; ++i)
        if (sorted[i].key == sorted[i - 1].key) { free(sorted); return -1; }
    s_off[0] = d_off[0] = 0;
    table128_job j = {words, n, norb, sorted, s_off, d_off};
    par_for(n, 4, nthreads, count128_range, &j);
    for (i64 i = 0; i < n; ++i) { s_off[i + 1] += s_off[i]; d_off[i + 1] += d_off[i]; }
    free(sorted);
    return 0;
}

void orc_table128_fill(const u64 *words, i64 n, int norb, const i64 *s_off, const i64 *d_off,
                       i64 *s_tgt, int16_t *s_hole, int16_t *s_part, int8_t *s_phase,
                       i64 *d_tgt, int16_t *d_h1, int16_t *d_h2, int16_t *d_p1, int16_t *d_p2, int8_t *d_phase,
                       int nthreads) {
    keyidx128 *sorted = make_sorted128(words, n);
    table128_job j = {words, n, norb, sorted, (i64 *)s_off, (i64 *)d_off, s_tgt, s_hole, s_part, s_phase,
                      d_tgt, d_h1, d_h2, d_p1, d_p2, d_phase};
    par_for(n, 4, nthreads, fill128_range, &j);
    free(sorted);
}

/* davidson.py:86-124: cyclic Jacobi on a symmetric n x n (row-major a, v). */
int orc_jacobi_kernel(double *a, double *v, int n, double tol, int max_sweeps) {
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) off += 2.0 * a[p * n + q] * a[p * n + q];
        if (sqrt(off) <= tol) return sweep;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                double apq = a[p * n + q];
                if (apq == 0.0) continue;
                double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
                double t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
                if (theta < 0.0) t = -t;
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                a[p * n + p] -= t * apq;
                a[q * n + q] += t * apq;
                a[p * n + q] = a[q * n + p] = 0.0;
                for (int k = 0; k < n; ++k) {
                    if (k == p || k == q) continue;
                    double akp = a[k * n + p], akq = a[k * n + q];
                    a[k * n + p] = c * akp - s * akq; a[p * n + k] = a[k * n + p];
                    a[k * n + q] = s * akp + c * akq; a[q * n + k] = a[k * n + q];
                }
                for (int k = 0; k < n; ++k) {
                    double vkp = v[k * n + p], vkq = v[k * n + q];
                    v[k * n + p] = c * vkp - s * vkq;
                    v[k * n + q] = s * vkp + c * vkq;
                }
            }
    }
    return max_sweeps;
}
