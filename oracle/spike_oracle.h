/*
 * spike_oracle.h — CPU restatement of the reference recursive-SPIKE path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1811_03559_b200/)
 * links, loads or calls this; only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may use it, and only as the
 * checker.  Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).  Parity of this restatement is
 * pinned against the compiled reference (oracle/_ref, built from the
 * reference sources by oracle/Makefile) through the fixtures in tests/golden/.
 *
 * Storage conventions follow the reference: band column-major with
 * ld = kl+ku+1, entry (i,j) at data[j*ld + ku+i-j] (banded_matrix.hpp:61-63);
 * dense blocks column-major.
 *
 * Generalisation beyond the reference: the reduced hierarchy accepts any
 * partition count p >= 1 (an odd unit at a level is carried unchanged to the
 * next level); for power-of-two p it is exactly the reference hierarchy.
 */
#ifndef SPIKE_ORACLE_H
#define SPIKE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_FIRSTLAST = 0, ORC_INNER_SINGLE = 1, ORC_INNER_DUAL = 2 };

typedef struct orc_plan {
    int p;
    int *bounds; /* p+1 */
    int *kinds;  /* p */
    int threads_used, idle_threads;
    double r12, r13;
} orc_plan;

typedef struct orc_fact orc_fact;

/* partition.cpp:47-54 */
void orc_compute_ratios(double kconst, int nrhs, int k, double *r12, double *r13);
/* partition.cpp:24-45, :56-87, :89-118 ; returns 0 or -1 (invalid t) */
int orc_make_plan(int n, int kl, int ku, int t, double r12, double r13, orc_plan *out);
/* plan from explicit bounds (any p >= 1; inner partitions single) */
int orc_plan_from_bounds(int p, const int *bounds, orc_plan *out);
void orc_plan_free(orc_plan *pl);

/* factorize.cpp:133-257 ; returns NULL on error (message via orc_last_error) */
orc_fact *orc_factorize(const double *band, int n, int kl, int ku, const orc_plan *plan,
                        int pivoting, double boost_eps);
void orc_fact_free(orc_fact *f);
int orc_fact_p(const orc_fact *f);
int orc_fact_k(const orc_fact *f);
int orc_fact_boost_count(const orc_fact *f);
int orc_fact_levels(const orc_fact *f);
void orc_fact_factor_sweeps(const orc_fact *f, long *out /* p */);
/* which: 0 vt, 1 vb, 2 wt, 3 wb, 4 bhat, 5 chat ; out k*k column-major */
void orc_fact_tip(const orc_fact *f, int which, int i, double *out);

/* solve.cpp:81-223 / :225-380 ; X is n x nrhs column-major (ld n) */
int orc_solve(const orc_fact *f, const double *F, int nrhs, int transpose, double *X,
              long *partition_sweeps /* p or NULL */, long *couplings /* or NULL */);

/* solve.cpp:382-402 over the reduced system built by reduce_factorize
 * (factorize.cpp:46-120) from explicit tips; z is 2pk x ncols, in place. */
int orc_reduced_solve_tips(const double *vt, const double *vb, const double *wt,
                           const double *wb, int p, int k, double *z, int ncols, int transpose,
                           long *couplings);

/* oracle.cpp:17-121 : serial padded-band GE (divides by the pivot) */
int orc_oracle_solve(const double *band, int n, int kl, int ku, const double *F, int nrhs,
                     int transpose, int pivoting, double *X);
/* oracle.cpp:132-166 */
double orc_condition_estimate_1norm(const double *band, int n, int kl, int ku);
/* band_ops.cpp:11-37 */
void orc_band_matmul(const double *band, int n, int kl, int ku, const double *X, int ncols,
                     int transpose, double *Y);
/* band_ops.cpp:45-57 (Frobenius) */
double orc_relative_residual(const double *band, int n, int kl, int ku, const double *X,
                             const double *F, int ncols, int transpose);
/* max_c ||A x_c - f_c||_inf / (||A||_inf ||x_c||_inf) */
double orc_backward_error_inf(const double *band, int n, int kl, int ku, const double *X,
                              const double *F, int ncols, int transpose);

/* BASELINE generator (include/spike_b200_gen.h) into a band / dense block */
void orc_generate_band(uint64_t seed, int n, int kl, int ku, double dd, double *band);
void orc_generate_rhs(uint64_t seed, int n, int ncols, double *F);

const char *orc_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
