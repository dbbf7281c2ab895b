/*
 * spike_oracle.c — CPU restatement of the reference recursive-SPIKE solver.
 *
 * TEST INFRASTRUCTURE ONLY (see spike_oracle.h).  Plain serial C: each
 * partition is processed in turn; the reference's InnerDual partitions
 * (two threads on a 2x2 split, spike2x2.cpp) produce mathematically the same
 * tips as a single-thread partition, so they are restated as single ones.
 * Citations are relative to /root/reference/proj.
 */
#include "spike_oracle.h"

#include "../include/spike_b200_gen.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
static void set_err(const char *m) { snprintf(g_err, sizeof g_err, "%s", m); }
const char *orc_last_error(void) { return g_err; }

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }

/* ----- band access (banded_matrix.hpp:41-50, :61-63) ----- */
static double band_at(const double *a, int n, int kl, int ku, int i, int j) {
    if (i < 0 || j < 0 || i >= n || j >= n) return 0.0;
    if (i - j > kl || j - i > ku) return 0.0;
    return a[(size_t)j * (kl + ku + 1) + (size_t)(ku + i - j)];
}

/* ----- planning (partition.cpp) ----- */
void orc_compute_ratios(double kc, int nrhs, int k, double *r12, double *r13) {
    /* partition.cpp:47-54 */
    const double rho = (double)nrhs / k;
    const double t = 1.0 / (1.0 + kc * rho) + (1.5 + 2.0 * rho) / (1.0 / kc + rho);
    *r13 = t;
    *r12 = t / 2.0;
}

static void distribute(int t, int cap, orc_plan *pl) {
    /* partition.cpp:24-45 */
    int p = 1;
    while (2 * p <= t) p *= 2;
    if (cap > 0 && cap < p) p = cap;
    pl->p = p;
    pl->kinds = (int *)calloc((size_t)p, sizeof(int));
    for (int i = 0; i < p; ++i) pl->kinds[i] = ORC_INNER_SINGLE;
    if (p == 1) {
        pl->kinds[0] = ORC_FIRSTLAST;
        pl->threads_used = 1;
        pl->idle_threads = t - 1;
        return;
    }
    pl->kinds[0] = pl->kinds[p - 1] = ORC_FIRSTLAST;
    const int extra = imin(t - p, p - 2);
    for (int i = 0; i < extra; ++i) pl->kinds[1 + i] = ORC_INNER_DUAL;
    pl->threads_used = p + extra;
    pl->idle_threads = t - pl->threads_used;
}

static int sizes_for(int n, const orc_plan *pl, double r12, double r13, int min_single,
                     int min_dual, int *sizes) {
    /* partition.cpp:56-87 ; -1 is the reference's domain_error */
    const int p = pl->p;
    if (p == 1) {
        if (n < min_single) return -1;
        sizes[0] = n;
        return 0;
    }
    int x = 0;
    for (int i = 0; i < p; ++i) x += pl->kinds[i] == ORC_INNER_DUAL;
    const int y = (p - x) - 2;
    const double denom = 2.0 * r12 * r13 + x * r13 + y * r12;
    const double n1 = n * r12 * r13 / denom, n2 = n1 / r12, n3 = n1 / r13;
    long long rest = 0;
    for (int i = 1; i < p; ++i) {
        double want = n1;
        if (pl->kinds[i] == ORC_INNER_DUAL) want = n2;
        else if (pl->kinds[i] == ORC_INNER_SINGLE) want = n3;
        sizes[i] = (int)llround(want);
        rest += sizes[i];
    }
    sizes[0] = (int)(n - rest);
    for (int i = 0; i < p; ++i) {
        const int need = pl->kinds[i] == ORC_INNER_DUAL ? min_dual : min_single;
        if (sizes[i] < need) return -1;
    }
    return 0;
}

int orc_make_plan(int n, int kl, int ku, int t, double r12, double r13, orc_plan *out) {
    /* partition.cpp:89-118 */
    memset(out, 0, sizeof *out);
    if (t < 1) {
        set_err("distribute_threads: t must be >= 1");
        return -1;
    }
    const int khat = imax(kl, ku);
    const int min_single = 2 * khat + 1;
    const int min_dual = imax(min_single, 2 * (kl + ku + 1));
    orc_plan base;
    distribute(t, 0, &base);
    for (int p = base.p; p >= 1; p /= 2) {
        orc_plan pl;
        memset(&pl, 0, sizeof pl);
        distribute(t, p, &pl);
        int *sizes = (int *)calloc((size_t)pl.p, sizeof(int));
        if (sizes_for(n, &pl, r12, r13, min_single, min_dual, sizes) == 0) {
            pl.bounds = (int *)calloc((size_t)pl.p + 1, sizeof(int));
            for (int i = 0; i < pl.p; ++i) pl.bounds[i + 1] = pl.bounds[i] + sizes[i];
            pl.r12 = r12;
            pl.r13 = r13;
            free(sizes);
            free(base.kinds);
            *out = pl;
            return 0;
        }
        free(sizes);
        free(pl.kinds);
        if (p == 1) break;
    }
    free(base.kinds);
    out->p = 1;
    out->kinds = (int *)calloc(1, sizeof(int));
    out->bounds = (int *)calloc(2, sizeof(int));
    out->bounds[1] = n;
    out->threads_used = 1;
    out->idle_threads = t - 1;
    out->r12 = r12;
    out->r13 = r13;
    return 0;
}

int orc_plan_from_bounds(int p, const int *bounds, orc_plan *out) {
    memset(out, 0, sizeof *out);
    if (p < 1) return -1;
    out->p = p;
    out->bounds = (int *)malloc(sizeof(int) * (size_t)(p + 1));
    memcpy(out->bounds, bounds, sizeof(int) * (size_t)(p + 1));
    out->kinds = (int *)malloc(sizeof(int) * (size_t)p);
    for (int i = 0; i < p; ++i) out->kinds[i] = (i == 0 || i == p - 1) ? ORC_FIRSTLAST : ORC_INNER_SINGLE;
    out->threads_used = p;
    out->r12 = 1.0;
    out->r13 = 2.0;
    return 0;
}

void orc_plan_free(orc_plan *pl) {
    free(pl->bounds);
    free(pl->kinds);
    pl->bounds = NULL;
    pl->kinds = NULL;
}

/* ----- per-partition band LU (kernels.cpp:29-118) ----- */
typedef struct {
    int n, kl, ku, ubw, d, rows, piv_on, boost_count;
    double *band;
    int *piv;
} lu_t;

#define LCOL(f, j) ((f)->band + (size_t)(j) * (f)->rows)

static int lu_factor_inplace(lu_t *f, double boost_eps) {
    /* kernels.cpp:79-118 */
    const int m = f->n;
    double amax = 0.0;
    for (size_t t = 0; t < (size_t)f->rows * m; ++t) amax = fmax(amax, fabs(f->band[t]));
    const double scale = amax == 0.0 ? 1.0 : amax;
    const double thresh = DBL_EPSILON * scale, bmag = boost_eps * scale;
    for (int j = 0; j < m; ++j) {
        double *cj = LCOL(f, j);
        const int rl = imin(f->kl, m - 1 - j);
        if (f->piv_on) {
            int ip = j;
            double best = fabs(cj[f->d]);
            for (int r = 1; r <= rl; ++r)
                if (fabs(cj[f->d + r]) > best) {
                    best = fabs(cj[f->d + r]);
                    ip = j + r;
                }
            if (best == 0.0) {
                set_err("lu_factor: exactly singular column in pivoting mode");
                return -2;
            }
            f->piv[j] = ip;
            if (ip != j) {
                const int ce = imin(m - 1, j + f->ubw);
                for (int c = j; c <= ce; ++c) {
                    double *cc = LCOL(f, c);
                    const double tmp = cc[f->d + j - c];
                    cc[f->d + j - c] = cc[f->d + ip - c];
                    cc[f->d + ip - c] = tmp;
                }
            }
        } else if (fabs(cj[f->d]) < thresh) {
            cj[f->d] = cj[f->d] == 0.0 ? bmag : copysign(bmag, cj[f->d]);
            f->boost_count++;
        }
        if (rl == 0) continue;
        const double inv = 1.0 / cj[f->d];
        for (int r = 1; r <= rl; ++r) cj[f->d + r] *= inv;
        const int ce = imin(m - 1, j + f->ubw);
        for (int c = j + 1; c <= ce; ++c) {
            double *cc = LCOL(f, c);
            const double ajc = cc[f->d + j - c];
            if (ajc == 0.0) continue;
            for (int r = 1; r <= rl; ++r) cc[f->d + j - c + r] -= ajc * cj[f->d + r];
        }
    }
    return 0;
}

/* kernels.cpp:29-65 : copy of A[r0..r0+m) (rows and columns reversed when rev) */
static int lu_init(lu_t *f, const double *a, int an, int akl, int aku, int r0, int m, int piv_on,
                   double boost_eps, int rev) {
    memset(f, 0, sizeof *f);
    f->n = m;
    f->kl = imin(rev ? aku : akl, m - 1);
    f->ku = imin(rev ? akl : aku, m - 1);
    f->piv_on = piv_on;
    f->ubw = piv_on ? imin(f->kl + f->ku, m - 1) : f->ku;
    f->d = f->ubw;
    f->rows = f->ubw + f->kl + 1;
    f->band = (double *)calloc((size_t)f->rows * m, sizeof(double));
    f->piv = (int *)malloc(sizeof(int) * (size_t)m);
    for (int j = 0; j < m; ++j) f->piv[j] = j;
    for (int j = 0; j < m; ++j)
        for (int i = imax(0, j - f->ku); i <= imin(m - 1, j + f->kl); ++i) {
            const int gi = rev ? r0 + m - 1 - i : r0 + i;
            const int gj = rev ? r0 + m - 1 - j : r0 + j;
            LCOL(f, j)[f->d + i - j] = band_at(a, an, akl, aku, gi, gj);
        }
    return lu_factor_inplace(f, boost_eps);
}

static void lu_free(lu_t *f) {
    free(f->band);
    free(f->piv);
    f->band = NULL;
    f->piv = NULL;
}

/* dense square block as a full band, pivoted with a boosted fallback
 * (kernels.cpp:67-77) */
static void lu_dense(lu_t *f, const double *m, int nn, double boost_eps, int *fell_back) {
    const int kb = imax(nn - 1, 0), ld = 2 * kb + 1;
    double *b = (double *)calloc((size_t)ld * nn, sizeof(double));
    for (int j = 0; j < nn; ++j)
        for (int i = 0; i < nn; ++i) b[(size_t)j * ld + kb + i - j] = m[(size_t)j * nn + i];
    *fell_back = 0;
    if (lu_init(f, b, nn, kb, kb, 0, nn, 1, boost_eps, 0) != 0) {
        lu_free(f);
        lu_init(f, b, nn, kb, kb, 0, nn, 0, boost_eps, 0);
        *fell_back = 1;
    }
    free(b);
}

#define BA(B, ld, i, c) ((B)[(size_t)(c) * (ld) + (i)])

static void swap_rows(double *B, int ld, int nc, int r1, int r2) {
    for (int c = 0; c < nc; ++c) {
        const double t = BA(B, ld, r1, c);
        BA(B, ld, r1, c) = BA(B, ld, r2, c);
        BA(B, ld, r2, c) = t;
    }
}

/* kernels.cpp:131-148 ; tail variant kernels.cpp:150-165 via row offset `off`
 * (B row r holds system row r+off, rows above off implicitly zero) */
static void fwd_lower(const lu_t *f, double *B, int ld, int nc, int start, int off) {
    for (int j = start; j < f->n; ++j) {
        if (f->piv_on && f->piv[j] != j) swap_rows(B, ld, nc, j - off, f->piv[j] - off);
        const int rl = imin(f->kl, f->n - 1 - j);
        if (rl == 0) continue;
        const double *lj = LCOL(f, j) + f->d + 1;
        for (int c = 0; c < nc; ++c) {
            const double bj = BA(B, ld, j - off, c);
            if (bj == 0.0) continue;
            for (int r = 0; r < rl; ++r) BA(B, ld, j - off + 1 + r, c) -= bj * lj[r];
        }
    }
}

/* kernels.cpp:167-183 */
static void bwd_upper(const lu_t *f, double *B, int ld, int nc, int begin) {
    for (int j = begin; j >= 0; --j) {
        const double ujj = LCOL(f, j)[f->d];
        const int ul = imin(f->ubw, j);
        const double *uj = LCOL(f, j) + f->d - ul;
        for (int c = 0; c < nc; ++c) {
            const double z = BA(B, ld, j, c) / ujj;
            BA(B, ld, j, c) = z;
            if (ul && z != 0.0)
                for (int r = 0; r < ul; ++r) BA(B, ld, j - ul + r, c) -= z * uj[r];
        }
    }
}

/* kernels.cpp:185-202 : bottom r rows of U^-1 B from B's bottom rows only.
 * B has `brows` rows whose last row is system row n-1. */
static void upper_bottom_tip(const lu_t *f, const double *B, int ld, int brows, int nc, int r,
                             double *T /* r x nc, ld r */) {
    r = imin(r, brows);
    const int off = f->n - r;
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < r; ++i) BA(T, r, i, c) = BA(B, ld, brows - r + i, c);
    for (int j = f->n - 1; j >= off; --j) {
        const double ujj = LCOL(f, j)[f->d];
        const int je = imin(f->n - 1, j + f->ubw);
        for (int c = 0; c < nc; ++c) {
            double s = BA(T, r, j - off, c);
            for (int j2 = j + 1; j2 <= je; ++j2) s -= LCOL(f, j2)[f->d + j - j2] * BA(T, r, j2 - off, c);
            BA(T, r, j - off, c) = s / ujj;
        }
    }
}

/* kernels.cpp:204-217 */
static void fwd_upperT(const lu_t *f, double *B, int ld, int nc) {
    for (int i = 0; i < f->n; ++i) {
        const int ul = imin(f->ubw, i);
        const double *ui = LCOL(f, i) + f->d - ul;
        const double uii = LCOL(f, i)[f->d];
        for (int c = 0; c < nc; ++c) {
            double s = BA(B, ld, i, c);
            for (int q = 0; q < ul; ++q) s -= ui[q] * BA(B, ld, i - ul + q, c);
            BA(B, ld, i, c) = s / uii;
        }
    }
}

/* kernels.cpp:219-234 (rows [lo, n) only; lo = 0 is the full sweep).  With
 * lo > 0 it is the windowed pass of lowerT_perm_bottom_tip (kernels.cpp:236-261):
 * B row r holds system row r+lo. */
static void bwd_lowerT(const lu_t *f, double *B, int ld, int nc, int lo) {
    for (int i = f->n - 1; i >= lo; --i) {
        const int rl = imin(f->kl, f->n - 1 - i);
        if (rl > 0) {
            const double *li = LCOL(f, i) + f->d + 1;
            for (int c = 0; c < nc; ++c) {
                double s = 0.0;
                for (int r = 0; r < rl; ++r) s += li[r] * BA(B, ld, i - lo + 1 + r, c);
                BA(B, ld, i - lo, c) -= s;
            }
        }
        if (f->piv_on && f->piv[i] != i) swap_rows(B, ld, nc, i - lo, f->piv[i] - lo);
    }
}

/* kernels.cpp:236-261 */
static void lowerT_perm_bottom_tip(const lu_t *f, const double *B, int ld, int nc, int r,
                                   double *T /* r x nc */) {
    r = imin(r, f->n);
    const int w = imin(f->n, r + (f->piv_on ? f->kl : 0));
    const int off = f->n - w;
    double *t = (double *)malloc(sizeof(double) * (size_t)w * (nc > 0 ? nc : 1));
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < w; ++i) BA(t, w, i, c) = BA(B, ld, off + i, c);
    bwd_lowerT(f, t, w, nc, off);
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < r; ++i) BA(T, r, i, c) = BA(t, w, w - r + i, c);
    free(t);
}

/* kernels.cpp:263-280 : B[n-r:] += (U[n-r:, n-r:])^-T T */
static void add_upperT_tail(const lu_t *f, double *B, int ld, int nc, const double *T, int r) {
    if (r == 0) return;
    const int off = f->n - r;
    double *z = (double *)calloc((size_t)r * (nc > 0 ? nc : 1), sizeof(double));
    for (int i = off; i < f->n; ++i) {
        const int ul = imin(f->ubw, i - off);
        const double uii = LCOL(f, i)[f->d];
        for (int c = 0; c < nc; ++c) {
            double s = BA(T, r, i - off, c);
            for (int j = i - ul; j < i; ++j) s -= LCOL(f, i)[f->d + j - i] * BA(z, r, j - off, c);
            BA(z, r, i - off, c) = s / uii;
        }
    }
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < r; ++i) BA(B, ld, off + i, c) += BA(z, r, i, c);
    free(z);
}

static int trunc_start(const lu_t *f, int corner) {
    /* block_util.hpp:13-16 */
    return imax(0, f->n - corner - (f->piv_on ? f->kl : 0));
}

static void reverse_rows(double *B, int ld, int rows, int nc) {
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < rows / 2; ++i) {
            const double t = BA(B, ld, i, c);
            BA(B, ld, i, c) = BA(B, ld, rows - 1 - i, c);
            BA(B, ld, rows - 1 - i, c) = t;
        }
}

/* C (r x nc) -= A (r x kk) * B (kk x nc) ; banded_matrix.cpp:39-44 */
static void gemm_minus(double *C, int ldc, const double *A, int lda, const double *B, int ldb,
                       int r, int kk, int nc) {
    for (int j = 0; j < nc; ++j)
        for (int l = 0; l < kk; ++l) {
            const double b = BA(B, ldb, l, j);
            if (b == 0.0) continue;
            for (int i = 0; i < r; ++i) BA(C, ldc, i, j) -= b * BA(A, lda, i, l);
        }
}

/* C (r x nc) -= A^T B, A is kk x r ; banded_matrix.cpp:46-51 */
static void gemm_minus_t(double *C, int ldc, const double *A, int lda, const double *B, int ldb,
                         int r, int kk, int nc) {
    for (int j = 0; j < nc; ++j)
        for (int i = 0; i < r; ++i) {
            double s = 0.0;
            for (int l = 0; l < kk; ++l) s += BA(A, lda, l, i) * BA(B, ldb, l, j);
            BA(C, ldc, i, j) -= s;
        }
}

/* out (r x nc) = A (r x kk) * B (kk x nc) */
static void gemm_set(double *C, int ldc, const double *A, int lda, const double *B, int ldb, int r,
                     int kk, int nc) {
    for (int j = 0; j < nc; ++j)
        for (int i = 0; i < r; ++i) BA(C, ldc, i, j) = 0.0;
    gemm_minus(C, ldc, A, lda, B, ldb, r, kk, nc);
    for (int j = 0; j < nc; ++j)
        for (int i = 0; i < r; ++i) BA(C, ldc, i, j) = -BA(C, ldc, i, j);
}

static void lu_solve(const lu_t *f, double *B, int ld, int nc, int transpose) {
    /* kernels.cpp:282-290 */
    if (!transpose) {
        fwd_lower(f, B, ld, nc, 0, 0);
        bwd_upper(f, B, ld, nc, f->n - 1);
    } else {
        fwd_upperT(f, B, ld, nc);
        bwd_lowerT(f, B, ld, nc, 0);
    }
}

/* ----- reduced hierarchy (factorize.hpp:26-49, factorize.cpp:19-120) ----- */
typedef struct {
    int p, k, L;
    int *units;   /* [L+1] */
    int **uoff;   /* [L+1][units] tip-row offsets */
    int **uh;     /* [L+1][units] heights */
    double ***v;  /* [L][units] h x k (NULL where never formed) */
    double ***w;
    lu_t **pairs; /* [L][units/2] */
    int boost_warnings;
} red_t;

static void pair_solve(const red_t *R, int l, int a, double *z, int ld, int nc) {
    /* factorize.cpp:19-32 */
    const int k = R->k, hL = R->uh[l][2 * a], hR = R->uh[l][2 * a + 1];
    const double *vl = R->v[l][2 * a], *wr = R->w[l][2 * a + 1];
    double *red = (double *)malloc(sizeof(double) * (size_t)2 * k * (nc > 0 ? nc : 1));
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < 2 * k; ++i) BA(red, 2 * k, i, c) = BA(z, ld, hL - k + i, c);
    lu_solve(&R->pairs[l][a], red, 2 * k, nc, 0);
    gemm_minus(z, ld, vl, hL, red + k, 2 * k, hL - k, k, nc);
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < 2 * k; ++i) BA(z, ld, hL - k + i, c) = BA(red, 2 * k, i, c);
    gemm_minus(z + hL + k, ld, wr + k, hR, red, 2 * k, hR - k, k, nc);
    free(red);
}

static void pair_solve_transpose(const red_t *R, int l, int a, double *z, int ld, int nc) {
    /* factorize.cpp:34-44 */
    const int k = R->k, hL = R->uh[l][2 * a], hR = R->uh[l][2 * a + 1];
    const double *vl = R->v[l][2 * a], *wr = R->w[l][2 * a + 1];
    double *red = (double *)malloc(sizeof(double) * (size_t)2 * k * (nc > 0 ? nc : 1));
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < 2 * k; ++i) BA(red, 2 * k, i, c) = BA(z, ld, hL - k + i, c);
    gemm_minus_t(red, 2 * k, wr + k, hR, z + hL + k, ld, k, hR - k, nc);
    gemm_minus_t(red + k, 2 * k, vl, hL, z, ld, k, hL - k, nc);
    lu_solve(&R->pairs[l][a], red, 2 * k, nc, 1);
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < 2 * k; ++i) BA(z, ld, hL - k + i, c) = BA(red, 2 * k, i, c);
    free(red);
}

static void red_build(red_t *R, const double *vt, const double *vb, const double *wt,
                      const double *wb, int p, int k, double boost_eps) {
    /* factorize.cpp:46-120, generalised to any p by carrying an odd unit */
    memset(R, 0, sizeof *R);
    R->p = p;
    R->k = k;
    if (p < 2 || k == 0) return;
    int L = 0;
    for (int u = p; u > 1; u = (u + 1) / 2) ++L;
    R->L = L;
    R->units = (int *)calloc((size_t)L + 1, sizeof(int));
    R->uoff = (int **)calloc((size_t)L + 1, sizeof(int *));
    R->uh = (int **)calloc((size_t)L + 1, sizeof(int *));
    R->v = (double ***)calloc((size_t)L + 1, sizeof(double **));
    R->w = (double ***)calloc((size_t)L + 1, sizeof(double **));
    R->pairs = (lu_t **)calloc((size_t)L, sizeof(lu_t *));
    R->units[0] = p;
    for (int l = 0; l <= L; ++l) {
        const int u = l == 0 ? p : (R->units[l - 1] + 1) / 2;
        R->units[l] = u;
        R->uoff[l] = (int *)calloc((size_t)u, sizeof(int));
        R->uh[l] = (int *)calloc((size_t)u, sizeof(int));
        R->v[l] = (double **)calloc((size_t)u, sizeof(double *));
        R->w[l] = (double **)calloc((size_t)u, sizeof(double *));
        for (int a = 0; a < u; ++a) {
            if (l == 0) {
                R->uoff[0][a] = 2 * a * k;
                R->uh[0][a] = 2 * k;
            } else if (2 * a + 1 < R->units[l - 1]) {
                R->uoff[l][a] = R->uoff[l - 1][2 * a];
                R->uh[l][a] = R->uh[l - 1][2 * a] + R->uh[l - 1][2 * a + 1];
            } else {
                R->uoff[l][a] = R->uoff[l - 1][2 * a];
                R->uh[l][a] = R->uh[l - 1][2 * a];
            }
        }
    }
    const size_t kk = (size_t)k * k;
    for (int i = 0; i < p; ++i) {
        if (i < p - 1) {
            double *col = (double *)calloc(2 * kk, sizeof(double));
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < k; ++r) {
                    BA(col, 2 * k, r, c) = vt[i * kk + (size_t)c * k + r];
                    BA(col, 2 * k, k + r, c) = vb[i * kk + (size_t)c * k + r];
                }
            R->v[0][i] = col;
        }
        if (i > 0) {
            double *col = (double *)calloc(2 * kk, sizeof(double));
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < k; ++r) {
                    BA(col, 2 * k, r, c) = wt[i * kk + (size_t)c * k + r];
                    BA(col, 2 * k, k + r, c) = wb[i * kk + (size_t)c * k + r];
                }
            R->w[0][i] = col;
        }
    }
    for (int l = 0; l < L; ++l) {
        const int units = R->units[l], np = units / 2;
        R->pairs[l] = (lu_t *)calloc((size_t)np, sizeof(lu_t));
        for (int a = 0; a < np; ++a) {
            const int hL = R->uh[l][2 * a], hR = R->uh[l][2 * a + 1];
            const double *vl = R->v[l][2 * a], *wr = R->w[l][2 * a + 1];
            double *cpl = (double *)calloc(4 * kk, sizeof(double));
            for (int i = 0; i < 2 * k; ++i) BA(cpl, 2 * k, i, i) = 1.0;
            for (int j = 0; j < k; ++j)
                for (int i = 0; i < k; ++i) {
                    BA(cpl, 2 * k, i, k + j) = BA(vl, hL, hL - k + i, j);
                    BA(cpl, 2 * k, k + i, j) = BA(wr, hR, i, j);
                }
            int fb = 0;
            lu_dense(&R->pairs[l][a], cpl, 2 * k, boost_eps, &fb);
            R->boost_warnings += fb;
            free(cpl);
            if (l + 1 == L) continue;
            const int H = hL + hR;
            if (2 * a + 1 < units - 1) {
                double *rhs = (double *)calloc((size_t)H * k, sizeof(double));
                for (int c = 0; c < k; ++c)
                    for (int i = 0; i < hR; ++i) BA(rhs, H, hL + i, c) = BA(R->v[l][2 * a + 1], hR, i, c);
                pair_solve(R, l, a, rhs, H, k);
                R->v[l + 1][a] = rhs;
            }
            if (a > 0) {
                double *rhs = (double *)calloc((size_t)H * k, sizeof(double));
                for (int c = 0; c < k; ++c)
                    for (int i = 0; i < hL; ++i) BA(rhs, H, i, c) = BA(R->w[l][2 * a], hL, i, c);
                pair_solve(R, l, a, rhs, H, k);
                R->w[l + 1][a] = rhs;
            }
        }
        if (units % 2 == 1 && l + 1 < L) {
            /* carried unit: D^(l) is the identity there */
            const int h = R->uh[l][units - 1];
            double *col = (double *)malloc(sizeof(double) * (size_t)h * k);
            memcpy(col, R->w[l][units - 1], sizeof(double) * (size_t)h * k);
            R->w[l + 1][np] = col;
        }
    }
}

static void red_free(red_t *R) {
    if (!R->units) return;
    for (int l = 0; l <= R->L; ++l) {
        for (int a = 0; a < R->units[l]; ++a) {
            free(R->v[l][a]);
            free(R->w[l][a]);
        }
        free(R->v[l]);
        free(R->w[l]);
        free(R->uoff[l]);
        free(R->uh[l]);
        if (l < R->L) {
            for (int a = 0; a < R->units[l] / 2; ++a) lu_free(&R->pairs[l][a]);
            free(R->pairs[l]);
        }
    }
    free(R->v);
    free(R->w);
    free(R->uoff);
    free(R->uh);
    free(R->pairs);
    free(R->units);
}

static long red_solve(const red_t *R, double *z, int ld, int nc, int transpose) {
    /* solve.cpp:33-55 */
    long cnt = 0;
    if (!transpose) {
        for (int l = 0; l < R->L; ++l)
            for (int a = 0; a < R->units[l] / 2; ++a, ++cnt)
                pair_solve(R, l, a, z + R->uoff[l][2 * a], ld, nc);
    } else {
        for (int l = R->L - 1; l >= 0; --l)
            for (int a = 0; a < R->units[l] / 2; ++a, ++cnt)
                pair_solve_transpose(R, l, a, z + R->uoff[l][2 * a], ld, nc);
    }
    return cnt;
}

int orc_reduced_solve_tips(const double *vt, const double *vb, const double *wt,
                           const double *wb, int p, int k, double *z, int nc, int transpose,
                           long *couplings) {
    red_t R;
    red_build(&R, vt, vb, wt, wb, p, k, sqrt(DBL_EPSILON));
    const long c = red_solve(&R, z, 2 * p * k, nc, transpose);
    if (couplings) *couplings += c;
    red_free(&R);
    return 0;
}

/* ----- factorization (factorize.cpp:133-257) ----- */
struct orc_fact {
    int n, kl, ku, k, p, piv_on;
    int *bounds, *kinds;
    lu_t *lu; /* per partition; last partition holds the reversed (UL) factors */
    double *bhat, *chat, *vt, *vb, *wt, *wb; /* p * k*k each */
    long *fsweeps;
    int boost_count;
    red_t red;
};

static void corner(const double *a, int n, int kl, int ku, int r0, int c0, int k, double *out) {
    /* spike2x2.cpp:17-26 */
    for (int j = 0; j < k; ++j)
        for (int i = 0; i < k; ++i) BA(out, k, i, j) = band_at(a, n, kl, ku, r0 + i, c0 + j);
}

orc_fact *orc_factorize(const double *band, int n, int kl, int ku, const orc_plan *plan,
                        int piv_on, double boost_eps) {
    if (plan->bounds[plan->p] != n) {
        set_err("factorize: plan does not match matrix");
        return NULL;
    }
    for (int i = 0; i < plan->p; ++i)
        if (plan->bounds[i + 1] - plan->bounds[i] < 1) {
            set_err("factorize: empty partition");
            return NULL;
        }
    orc_fact *F = (orc_fact *)calloc(1, sizeof *F);
    const int p = plan->p, k = imax(kl, ku);
    const size_t kk = (size_t)k * k;
    F->n = n;
    F->kl = kl;
    F->ku = ku;
    F->k = k;
    F->p = p;
    F->piv_on = piv_on;
    F->bounds = (int *)malloc(sizeof(int) * (size_t)(p + 1));
    memcpy(F->bounds, plan->bounds, sizeof(int) * (size_t)(p + 1));
    F->kinds = (int *)malloc(sizeof(int) * (size_t)p);
    memcpy(F->kinds, plan->kinds, sizeof(int) * (size_t)p);
    F->lu = (lu_t *)calloc((size_t)p, sizeof(lu_t));
    double **blk[6] = {&F->bhat, &F->chat, &F->vt, &F->vb, &F->wt, &F->wb};
    for (int b = 0; b < 6; ++b) *blk[b] = (double *)calloc(kk * p + 1, sizeof(double));
    F->fsweeps = (long *)calloc((size_t)p, sizeof(long));
    for (int i = 0; i + 1 < p; ++i) {
        const int b = plan->bounds[i + 1];
        corner(band, n, kl, ku, b - k, b, k, F->bhat + i * kk);
        corner(band, n, kl, ku, b, b - k, k, F->chat + (i + 1) * kk);
    }
    for (int i = 0; i < p; ++i) {
        const int r0 = plan->bounds[i], m = plan->bounds[i + 1] - r0;
        const int last = (p > 1 && i == p - 1);
        lu_t *lu = &F->lu[i];
        if (lu_init(lu, band, n, kl, ku, r0, m, piv_on, boost_eps, last) != 0) {
            orc_fact_free(F);
            return NULL;
        }
        F->boost_count += lu->boost_count;
        if (p == 1 || k == 0) continue;
        if (i == 0 || last) {
            /* first: vb_0 ; last: wt_{p-1} in reversed space (factorize.cpp:215-235) */
            double *rhs = (double *)calloc((size_t)m * k, sizeof(double));
            const double *cn = last ? F->chat + i * kk : F->bhat;
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < k; ++r)
                    BA(rhs, m, m - k + r, c) = last ? BA(cn, k, k - 1 - r, c) : BA(cn, k, r, c);
            fwd_lower(lu, rhs, m, k, trunc_start(lu, k), 0);
            double *tip = (double *)malloc(sizeof(double) * kk);
            upper_bottom_tip(lu, rhs, m, m, k, k, tip);
            if (last) {
                reverse_rows(tip, k, k, k);
                memcpy(F->wt + i * kk, tip, sizeof(double) * kk);
            } else {
                memcpy(F->vb, tip, sizeof(double) * kk);
            }
            free(tip);
            free(rhs);
        } else {
            /* inner (single or dual): factorize.cpp:191-209 */
            double *vc = (double *)calloc((size_t)m * k, sizeof(double));
            double *wc = (double *)calloc((size_t)m * k, sizeof(double));
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < k; ++r) {
                    BA(vc, m, m - k + r, c) = BA(F->bhat + i * kk, k, r, c);
                    BA(wc, m, r, c) = BA(F->chat + i * kk, k, r, c);
                }
            fwd_lower(lu, vc, m, k, trunc_start(lu, k), 0);
            bwd_upper(lu, vc, m, k, m - 1);
            fwd_lower(lu, wc, m, k, 0, 0);
            bwd_upper(lu, wc, m, k, m - 1);
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < k; ++r) {
                    BA(F->vt + i * kk, k, r, c) = BA(vc, m, r, c);
                    BA(F->vb + i * kk, k, r, c) = BA(vc, m, m - k + r, c);
                    BA(F->wt + i * kk, k, r, c) = BA(wc, m, r, c);
                    BA(F->wb + i * kk, k, r, c) = BA(wc, m, m - k + r, c);
                }
            F->fsweeps[i] = 3;
            free(vc);
            free(wc);
        }
    }
    red_build(&F->red, F->vt, F->vb, F->wt, F->wb, p, k, boost_eps);
    return F;
}

void orc_fact_free(orc_fact *F) {
    if (!F) return;
    for (int i = 0; i < F->p; ++i) lu_free(&F->lu[i]);
    free(F->lu);
    free(F->bounds);
    free(F->kinds);
    free(F->bhat);
    free(F->chat);
    free(F->vt);
    free(F->vb);
    free(F->wt);
    free(F->wb);
    free(F->fsweeps);
    red_free(&F->red);
    free(F);
}

int orc_fact_p(const orc_fact *F) { return F->p; }
int orc_fact_k(const orc_fact *F) { return F->k; }
int orc_fact_boost_count(const orc_fact *F) { return F->boost_count; }
int orc_fact_levels(const orc_fact *F) { return F->red.L; }
void orc_fact_factor_sweeps(const orc_fact *F, long *out) {
    memcpy(out, F->fsweeps, sizeof(long) * (size_t)F->p);
}
void orc_fact_tip(const orc_fact *F, int which, int i, double *out) {
    const double *src[6] = {F->vt, F->vb, F->wt, F->wb, F->bhat, F->chat};
    const size_t kk = (size_t)F->k * F->k;
    memcpy(out, src[which] + i * kk, sizeof(double) * kk);
}

/* ----- solves (solve.cpp:81-380) ----- */
int orc_solve(const orc_fact *F, const double *Fr, int nrhs, int transpose, double *X,
              long *psweeps, long *couplings) {
    const int n = F->n, p = F->p, k = F->k;
    const size_t kk = (size_t)k * k;
    memcpy(X, Fr, sizeof(double) * (size_t)n * nrhs);
    if (psweeps) memset(psweeps, 0, sizeof(long) * (size_t)p);
    if (couplings) *couplings = 0;
    if (p == 1) {
        lu_solve(&F->lu[0], X, n, nrhs, transpose);
        if (psweeps) psweeps[0] = 2;
        return 0;
    }
    const int T = 2 * p * k;
    double *tips = (double *)calloc((size_t)T * (nrhs > 0 ? nrhs : 1), sizeof(double));
    /* transpose S-stage tips tau_t / tau_b: k x nrhs per partition */
    double *tau_t = (double *)calloc((size_t)k * (nrhs > 0 ? nrhs : 1) * p + 1, sizeof(double));
    double *tau_b = (double *)calloc((size_t)k * (nrhs > 0 ? nrhs : 1) * p + 1, sizeof(double));
    double *tmp = (double *)calloc((size_t)k * (nrhs > 0 ? nrhs : 1) + 1, sizeof(double));
    const size_t kn = (size_t)k * nrhs;
#define TIP_T(i) (tips + 2 * (size_t)(i) * k)
#define TIP_B(i) (tips + (2 * (size_t)(i) + 1) * k)
    if (!transpose) {
        for (int i = 0; i < p; ++i) {
            const int r0 = F->bounds[i], m = F->bounds[i + 1] - r0;
            const lu_t *lu = &F->lu[i];
            double *xi = X + r0;
            if (i == 0) {
                fwd_lower(lu, xi, n, nrhs, 0, 0);
                upper_bottom_tip(lu, xi, n, m, nrhs, k, tmp);
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < k; ++r) BA(TIP_B(0), T, r, c) = BA(tmp, k, r, c);
            } else if (i == p - 1) {
                reverse_rows(xi, n, m, nrhs);
                fwd_lower(lu, xi, n, nrhs, 0, 0);
                upper_bottom_tip(lu, xi, n, m, nrhs, k, tmp);
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < k; ++r) BA(TIP_T(i), T, r, c) = BA(tmp, k, k - 1 - r, c);
            } else {
                fwd_lower(lu, xi, n, nrhs, 0, 0);
                bwd_upper(lu, xi, n, nrhs, m - 1);
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < k; ++r) {
                        BA(TIP_T(i), T, r, c) = BA(xi, n, r, c);
                        BA(TIP_B(i), T, r, c) = BA(xi, n, m - k + r, c);
                    }
            }
            if (psweeps) psweeps[i] += (i == 0 || i == p - 1) ? 1 : 2;
        }
        const long cc = red_solve(&F->red, tips, T, nrhs, 0);
        if (couplings) *couplings = cc;
        for (int i = 0; i < p; ++i) {
            const int r0 = F->bounds[i], m = F->bounds[i + 1] - r0;
            const lu_t *lu = &F->lu[i];
            double *xi = X + r0;
            if (i == 0 || i == p - 1) {
                const int last = i == p - 1;
                const int s = trunc_start(lu, k);
                double *corr = (double *)calloc((size_t)(m - s) * (nrhs > 0 ? nrhs : 1), sizeof(double));
                if (!last) gemm_set(tmp, k, F->bhat, k, TIP_T(1), T, k, k, nrhs);
                else gemm_set(tmp, k, F->chat + i * kk, k, TIP_B(i - 1), T, k, k, nrhs);
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < k; ++r)
                        BA(corr, m - s, m - s - k + r, c) = last ? BA(tmp, k, k - 1 - r, c) : BA(tmp, k, r, c);
                fwd_lower(lu, corr, m - s, nrhs, s, s);
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < m - s; ++r) BA(xi, n, s + r, c) -= BA(corr, m - s, r, c);
                bwd_upper(lu, xi, n, nrhs, m - 1);
                if (last) reverse_rows(xi, n, m, nrhs);
                free(corr);
                if (psweeps) psweeps[i] += 1;
            } else {
                double *corr = (double *)calloc((size_t)m * (nrhs > 0 ? nrhs : 1), sizeof(double));
                gemm_set(corr, m, F->chat + i * kk, k, TIP_B(i - 1), T, k, k, nrhs);
                gemm_set(corr + m - k, m, F->bhat + i * kk, k, TIP_T(i + 1), T, k, k, nrhs);
                fwd_lower(lu, corr, m, nrhs, 0, 0);
                bwd_upper(lu, corr, m, nrhs, m - 1);
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < m; ++r) BA(xi, n, r, c) -= BA(corr, m, r, c);
                free(corr);
                if (psweeps) psweeps[i] += 2;
            }
        }
    } else {
        /* S stage (solve.cpp:248-309) */
        for (int i = 0; i < p; ++i) {
            const int r0 = F->bounds[i], m = F->bounds[i + 1] - r0;
            const lu_t *lu = &F->lu[i];
            if (i == 0 || i == p - 1) {
                const int last = i == p - 1;
                double *xi = X + r0;
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < k; ++r) BA(xi, n, last ? r : m - k + r, c) = 0.0;
                if (last) reverse_rows(xi, n, m, nrhs);
                fwd_upperT(lu, xi, n, nrhs);
                lowerT_perm_bottom_tip(lu, xi, n, nrhs, k, tmp);
                double *dst = last ? tau_t + (size_t)i * kn : tau_b + (size_t)i * kn;
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < k; ++r) BA(dst, k, r, c) = BA(tmp, k, last ? k - 1 - r : r, c);
                if (psweeps) psweeps[i] += 1;
            } else {
                double *v = (double *)malloc(sizeof(double) * (size_t)m * (nrhs > 0 ? nrhs : 1));
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < m; ++r)
                        BA(v, m, r, c) = (r < k || r >= m - k) ? 0.0 : BA(Fr + r0, n, r, c);
                fwd_upperT(lu, v, m, nrhs);
                bwd_lowerT(lu, v, m, nrhs, 0);
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < k; ++r) {
                        BA(tau_t + (size_t)i * kn, k, r, c) = BA(v, m, r, c);
                        BA(tau_b + (size_t)i * kn, k, r, c) = BA(v, m, m - k + r, c);
                    }
                free(v);
                if (psweeps) psweeps[i] += 2;
            }
        }
        /* G tips (solve.cpp:313-325) */
        for (int c = 0; c < nrhs; ++c)
            for (int r = 0; r < k; ++r) {
                BA(TIP_T(0), T, r, c) = BA(Fr, n, r, c);
                BA(TIP_B(p - 1), T, r, c) = BA(Fr, n, n - k + r, c);
            }
        for (int i = 1; i < p; ++i) {
            for (int c = 0; c < nrhs; ++c)
                for (int r = 0; r < k; ++r) BA(TIP_T(i), T, r, c) = BA(Fr, n, F->bounds[i] + r, c);
            gemm_minus_t(TIP_T(i), T, F->bhat + (i - 1) * kk, k, tau_b + (size_t)(i - 1) * kn, k, k, k, nrhs);
        }
        for (int i = 0; i + 1 < p; ++i) {
            for (int c = 0; c < nrhs; ++c)
                for (int r = 0; r < k; ++r) BA(TIP_B(i), T, r, c) = BA(Fr, n, F->bounds[i + 1] - k + r, c);
            gemm_minus_t(TIP_B(i), T, F->chat + (i + 1) * kk, k, tau_t + (size_t)(i + 1) * kn, k, k, k, nrhs);
        }
        const long cc = red_solve(&F->red, tips, T, nrhs, 1);
        if (couplings) *couplings = cc;
        /* D^T stage (solve.cpp:331-376) */
        for (int i = 0; i < p; ++i) {
            const int r0 = F->bounds[i], m = F->bounds[i + 1] - r0;
            const lu_t *lu = &F->lu[i];
            double *xi = X + r0;
            if (i == 0 || i == p - 1) {
                const int last = i == p - 1;
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < k; ++r)
                        BA(tmp, k, r, c) = last ? BA(TIP_T(i), T, k - 1 - r, c) : BA(TIP_B(0), T, r, c);
                add_upperT_tail(lu, xi, n, nrhs, tmp, k);
                bwd_lowerT(lu, xi, n, nrhs, 0);
                if (last) reverse_rows(xi, n, m, nrhs);
                if (psweeps) psweeps[i] += 1;
            } else {
                for (int c = 0; c < nrhs; ++c)
                    for (int r = 0; r < k; ++r) {
                        BA(xi, n, r, c) = BA(TIP_T(i), T, r, c);
                        BA(xi, n, m - k + r, c) = BA(TIP_B(i), T, r, c);
                    }
                fwd_upperT(lu, xi, n, nrhs);
                bwd_lowerT(lu, xi, n, nrhs, 0);
                if (psweeps) psweeps[i] += 2;
            }
        }
    }
#undef TIP_T
#undef TIP_B
    free(tips);
    free(tau_t);
    free(tau_b);
    free(tmp);
    return 0;
}

/* ----- serial banded GE oracle (oracle.cpp:17-121) ----- */
typedef struct {
    int n, kl, ku, ubw, d, rows, sign;
    double *ab;
    int *piv;
} bge_t;

static int bge_init(bge_t *g, const double *a, int n, int kl, int ku, int pivoting) {
    g->n = n;
    g->kl = kl;
    g->ku = ku;
    g->ubw = kl + ku;
    g->d = kl + ku;
    g->rows = 2 * kl + ku + 1;
    g->sign = 1;
    g->ab = (double *)calloc((size_t)g->rows * n, sizeof(double));
    g->piv = (int *)malloc(sizeof(int) * (size_t)n);
    for (int j = 0; j < n; ++j)
        for (int i = imax(0, j - ku); i <= imin(n - 1, j + kl); ++i)
            g->ab[(size_t)j * g->rows + g->d + i - j] = band_at(a, n, kl, ku, i, j);
    double amax = 0.0;
    for (size_t t = 0; t < (size_t)g->rows * n; ++t) amax = fmax(amax, fabs(g->ab[t]));
    const double scale = amax == 0.0 ? 1.0 : amax;
    const double zt = DBL_EPSILON * scale, bm = sqrt(DBL_EPSILON) * scale;
    for (int j = 0; j < n; ++j) {
        double *cj = g->ab + (size_t)j * g->rows;
        const int rl = imin(kl, n - 1 - j);
        int ip = j;
        if (pivoting) {
            double best = fabs(cj[g->d]);
            for (int r = 1; r <= rl; ++r)
                if (fabs(cj[g->d + r]) > best) {
                    best = fabs(cj[g->d + r]);
                    ip = j + r;
                }
            if (best == 0.0) {
                set_err("oracle_solve: singular matrix");
                return -2;
            }
            if (ip != j) {
                g->sign = -g->sign;
                for (int c = j; c <= imin(n - 1, j + g->ubw); ++c) {
                    double *cc = g->ab + (size_t)c * g->rows;
                    const double t = cc[g->d + j - c];
                    cc[g->d + j - c] = cc[g->d + ip - c];
                    cc[g->d + ip - c] = t;
                }
            }
        } else if (fabs(cj[g->d]) < zt) {
            cj[g->d] = cj[g->d] == 0.0 ? bm : copysign(bm, cj[g->d]);
        }
        g->piv[j] = ip;
        const double pv = cj[g->d];
        for (int r = 1; r <= rl; ++r) cj[g->d + r] /= pv;
        for (int c = j + 1; c <= imin(n - 1, j + g->ubw); ++c) {
            double *cc = g->ab + (size_t)c * g->rows;
            const double ajc = cc[g->d + j - c];
            if (ajc == 0.0) continue;
            for (int r = 1; r <= rl; ++r) cc[g->d + j + r - c] -= cj[g->d + r] * ajc;
        }
    }
    return 0;
}

static void bge_solve(const bge_t *g, double *x) {
    for (int j = 0; j < g->n; ++j) {
        if (g->piv[j] != j) {
            const double t = x[j];
            x[j] = x[g->piv[j]];
            x[g->piv[j]] = t;
        }
        const double *cj = g->ab + (size_t)j * g->rows;
        for (int r = 1; r <= imin(g->kl, g->n - 1 - j); ++r) x[j + r] -= cj[g->d + r] * x[j];
    }
    for (int j = g->n - 1; j >= 0; --j) {
        const double *cj = g->ab + (size_t)j * g->rows;
        x[j] /= cj[g->d];
        for (int r = 1; r <= imin(g->ubw, j); ++r) x[j - r] -= cj[g->d - r] * x[j];
    }
}

static void bge_free(bge_t *g) {
    free(g->ab);
    free(g->piv);
}

static double *band_transpose(const double *a, int n, int kl, int ku) {
    /* band_ops.cpp:77-85 : result has kl' = ku, ku' = kl */
    const int ld = kl + ku + 1;
    double *t = (double *)calloc((size_t)ld * n, sizeof(double));
    for (int j = 0; j < n; ++j)
        for (int i = imax(0, j - ku); i <= imin(n - 1, j + kl); ++i)
            t[(size_t)i * ld + (kl + j - i)] = band_at(a, n, kl, ku, i, j);
    return t;
}

int orc_oracle_solve(const double *band, int n, int kl, int ku, const double *F, int nrhs,
                     int transpose, int pivoting, double *X) {
    const double *a = band;
    double *at = NULL;
    if (transpose) {
        at = band_transpose(band, n, kl, ku);
        a = at;
        const int t = kl;
        kl = ku;
        ku = t;
    }
    bge_t g;
    const int rc = bge_init(&g, a, n, kl, ku, pivoting);
    if (rc == 0) {
        memcpy(X, F, sizeof(double) * (size_t)n * nrhs);
        for (int c = 0; c < nrhs; ++c) bge_solve(&g, X + (size_t)c * n);
    }
    bge_free(&g);
    free(at);
    return rc;
}

double orc_condition_estimate_1norm(const double *band, int n, int kl, int ku) {
    /* oracle.cpp:132-166 (Hager) */
    bge_t fw, bw;
    double *at = band_transpose(band, n, kl, ku);
    if (bge_init(&fw, band, n, kl, ku, 1) != 0 || bge_init(&bw, at, n, ku, kl, 1) != 0) {
        free(at);
        return INFINITY;
    }
    double *x = (double *)malloc(sizeof(double) * (size_t)n);
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    double *xi = (double *)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) x[i] = 1.0 / n;
    double est = 0.0;
    for (int it = 0; it < 6; ++it) {
        memcpy(y, x, sizeof(double) * (size_t)n);
        bge_solve(&fw, y);
        double yn = 0.0;
        for (int i = 0; i < n; ++i) yn += fabs(y[i]);
        est = fmax(est, yn);
        for (int i = 0; i < n; ++i) xi[i] = y[i] >= 0.0 ? 1.0 : -1.0;
        bge_solve(&bw, xi);
        int jmax = 0;
        double zmax = 0.0, zdx = 0.0;
        for (int i = 0; i < n; ++i) {
            zdx += xi[i] * x[i];
            if (fabs(xi[i]) > zmax) {
                zmax = fabs(xi[i]);
                jmax = i;
            }
        }
        if (zmax <= zdx) break;
        memset(x, 0, sizeof(double) * (size_t)n);
        x[jmax] = 1.0;
    }
    double n1 = 0.0;
    for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int i = imax(0, j - ku); i <= imin(n - 1, j + kl); ++i) s += fabs(band_at(band, n, kl, ku, i, j));
        n1 = fmax(n1, s);
    }
    bge_free(&fw);
    bge_free(&bw);
    free(at);
    free(x);
    free(y);
    free(xi);
    return est * n1;
}

void orc_band_matmul(const double *band, int n, int kl, int ku, const double *X, int nc,
                     int transpose, double *Y) {
    memset(Y, 0, sizeof(double) * (size_t)n * nc);
    for (int j = 0; j < n; ++j)
        for (int i = imax(0, j - ku); i <= imin(n - 1, j + kl); ++i) {
            const double a = band_at(band, n, kl, ku, i, j);
            for (int c = 0; c < nc; ++c) {
                if (!transpose) BA(Y, n, i, c) += a * BA(X, n, j, c);
                else BA(Y, n, j, c) += a * BA(X, n, i, c);
            }
        }
}

double orc_relative_residual(const double *band, int n, int kl, int ku, const double *X,
                             const double *F, int nc, int transpose) {
    double *r = (double *)malloc(sizeof(double) * (size_t)n * (nc > 0 ? nc : 1));
    orc_band_matmul(band, n, kl, ku, X, nc, transpose, r);
    double rn = 0.0, fn = 0.0;
    for (size_t t = 0; t < (size_t)n * nc; ++t) {
        rn += (r[t] - F[t]) * (r[t] - F[t]);
        fn += F[t] * F[t];
    }
    free(r);
    if (fn == 0.0) return rn == 0.0 ? 0.0 : INFINITY;
    return sqrt(rn) / sqrt(fn);
}

double orc_backward_error_inf(const double *band, int n, int kl, int ku, const double *X,
                              const double *F, int nc, int transpose) {
    double *r = (double *)malloc(sizeof(double) * (size_t)n * (nc > 0 ? nc : 1));
    orc_band_matmul(band, n, kl, ku, X, nc, transpose, r);
    double anorm = 0.0; /* ||A||_inf (or ||A^T||_inf = ||A||_1) */
    const int lo = transpose ? ku : kl, hi = transpose ? kl : ku; /* row i of op(A): j in [i-lo, i+hi] */
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = imax(0, i - lo); j <= imin(n - 1, i + hi); ++j)
            s += fabs(transpose ? band_at(band, n, kl, ku, j, i) : band_at(band, n, kl, ku, i, j));
        anorm = fmax(anorm, s);
    }
    double worst = 0.0;
    for (int c = 0; c < nc; ++c) {
        double rm = 0.0, xm = 0.0;
        for (int i = 0; i < n; ++i) {
            rm = fmax(rm, fabs(BA(r, n, i, c) - BA(F, n, i, c)));
            xm = fmax(xm, fabs(BA(X, n, i, c)));
        }
        if (xm > 0.0) worst = fmax(worst, rm / (anorm * xm));
    }
    free(r);
    return worst;
}

void orc_generate_band(uint64_t seed, int n, int kl, int ku, double dd, double *band) {
    const int ld = kl + ku + 1;
    memset(band, 0, sizeof(double) * (size_t)ld * n);
    for (int j = 0; j < n; ++j)
        for (int i = imax(0, j - ku); i <= imin(n - 1, j + kl); ++i)
            band[(size_t)j * ld + (ku + i - j)] = spk_gen_entry(seed, n, kl, ku, dd, i, j);
}

void orc_generate_rhs(uint64_t seed, int n, int nc, double *F) {
    for (int c = 0; c < nc; ++c)
        for (int i = 0; i < n; ++i) F[(size_t)c * n + i] = spk_gen_rhs(seed, i, c);
}
