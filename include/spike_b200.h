/*
 * spike_b200.h — C-ABI of the B200-native recursive SPIKE banded solver.
 *
 * This is the drop-in boundary under the reference's C++ solver API
 * (/root/reference/proj/include/spike/{factorize,solve,partition}.hpp).  Plain
 * pointers and sizes only; no exceptions, no torch types.  The C++ wrapper in
 * include/spike/*.hpp (namespace spike) maps the status codes back to the
 * reference's exception types.
 *
 * Entry point                reference interface it replaces
 * -------------------------  ------------------------------------------------
 * spk_factorize              spike::factorize            factorize.hpp:76-77
 * spk_solve (transpose=0/1)  spike::solve / transpose_solve  solve.hpp:23-29
 * spk_make_plan              spike::make_plan            partition.hpp:56
 * spk_compute_ratios         spike::compute_ratios       partition.hpp:45
 * spk_distribute_threads     spike::distribute_threads   partition.hpp:39
 * spk_compute_sizes          spike::compute_sizes        partition.hpp:51-52
 * spk_gpu_plan               (new) arbitrary-p planner mapped onto SMs
 * spk_fact_* getters         SpikeFactorization fields   factorize.hpp:56-74
 * spk_reduced_*              reduce_factorize / reduced_solve(_transpose)
 *                                                        factorize.hpp:45-49, solve.hpp:33-36
 * spk_band_matmul            spike::band_matmul          band_ops.hpp:11
 *
 * Memory: `band`, `F` and `X` may live on the host or on the device; say which
 * with SPK_MEM_HOST / SPK_MEM_DEVICE.  Host buffers are staged through the
 * call's stream (pinned host memory makes the copies asynchronous).  All work
 * is ordered on the stream passed in (NULL = the legacy default stream).
 * A factorization is immutable after spk_factorize returns and may be used by
 * any number of concurrent spk_solve calls on different streams.
 */
#ifndef SPIKE_B200_H
#define SPIKE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum spk_status {
    SPK_OK = 0,
    SPK_EINVAL = 1,    /* std::invalid_argument (shape / plan)          */
    SPK_ESINGULAR = 2, /* std::runtime_error (exactly singular column)  */
    SPK_EDOMAIN = 3,   /* std::domain_error (sizing)                    */
    SPK_ECUDA = 4,     /* CUDA runtime failure                          */
    SPK_ENOMEM = 5,    /* device allocation failure                     */
    SPK_ENCCL = 6,     /* collective failure                            */
    SPK_ERANGE = 7,    /* std::out_of_range                             */
    SPK_EIO = 8        /* std::runtime_error (file open / format, band_io.cpp) */
} spk_status;

enum { SPK_MEM_HOST = 0, SPK_MEM_DEVICE = 1 };
enum { SPK_FIRSTLAST = 0, SPK_INNER_SINGLE = 1, SPK_INNER_DUAL = 2 };
enum { SPK_TIP_VT = 0, SPK_TIP_VB = 1, SPK_TIP_WT = 2, SPK_TIP_WB = 3, SPK_BHAT = 4, SPK_CHAT = 5 };

typedef struct spk_fact spk_fact;
typedef struct spk_reduced spk_reduced;

/* Partition plan: p partitions, bounds[p+1] row offsets (bounds[0]=0,
 * bounds[p]=n), kinds[p] (informational on the GPU: dual partitions are
 * factored like single ones; the tips are the same mathematical objects). */
typedef struct spk_plan {
    int32_t p;
    const int64_t *bounds;
    const int32_t *kinds;
} spk_plan;

typedef struct spk_factor_options {
    int32_t pivoting;  /* FactorOptions::pivoting   (factorize.hpp:13-16) */
    double boost_eps;  /* FactorOptions::boost_eps  (<= 0 -> sqrt(eps))   */
} spk_factor_options;

const char *spk_last_error(void); /* thread-local message of the last failure */
const char *spk_version(void);

/* ---- planning (host-only, no GPU needed) ---- */
void spk_compute_ratios(double K, int32_t nrhs, int32_t k, double *r12, double *r13);
/* distribute_threads(t, cap_p): p and kinds[p] (kinds capacity >= p) */
spk_status spk_distribute_threads(int32_t t, int32_t cap_p, int32_t *p, int32_t *kinds,
                                  int32_t kinds_cap, int32_t *threads_used, int32_t *idle);
spk_status spk_compute_sizes(int64_t n, int32_t p, const int32_t *kinds, double r12, double r13,
                             int64_t min_single, int64_t min_dual, int64_t *sizes);
/* reference make_plan: bounds capacity >= p+1, kinds capacity >= p */
spk_status spk_make_plan(int64_t n, int32_t kl, int32_t ku, int32_t t, double r12, double r13,
                         int32_t cap, int32_t *p, int64_t *bounds, int32_t *kinds,
                         int32_t *threads_used, int32_t *idle);
/* B200 planner: p chosen for the GPU (any p >= 1, not only powers of two);
 * p_hint > 0 forces p.  First/last partitions sized by the reference ratio
 * model with K fitted to the device. */
spk_status spk_gpu_plan(int64_t n, int32_t kl, int32_t ku, int32_t nrhs, int32_t pivoting,
                        int32_t p_hint, int32_t cap, int32_t *p, int64_t *bounds,
                        int32_t *kinds);

/* ---- K calibration and ratio planning on the GPU (partition.cpp:120-170,
 * partition.hpp:58-74) ---- */
typedef struct spk_calibration {
    double k;              /* median over reps of t_solve(nrhs = k_sample) / t_factor */
    double factor_seconds; /* mean, one partition factorized on the GPU */
    double solve_seconds;  /* mean, its two-sweep solve */
    int32_t timer_warning; /* total sample < 10 ms (the reference's rule) */
} spk_calibration;
/* calibrate_k on the device: one non-pivoting partition of n_sample rows
 * (n_sample <= 0: 200 * k_sample) and bandwidth k_sample, CUDA-event timed. */
spk_status spk_calibrate_k(int64_t n_sample, int32_t k_sample, int32_t reps, void *stream,
                           spk_calibration *out);
/* default_k_cache_path (copied into buf, NUL-terminated): $SPIKE_K_CACHE or
 * "spike_k.cache"; write/read_k_cache in the reference's "K <value>" format.
 * spk_read_k_cache sets *found = 0 when the file or the key is missing. */
spk_status spk_default_k_cache_path(char *buf, int32_t cap);
spk_status spk_write_k_cache(const char *path, double k);
spk_status spk_read_k_cache(const char *path, double *k, int32_t *found);
/* spk_gpu_plan with explicit first/last partitions r13 x the inner size
 * (the reference's R13, partition.cpp:47-54; r12 has no GPU counterpart:
 * dual partitions factor like single ones). */
spk_status spk_gpu_plan_ratio(int64_t n, int32_t kl, int32_t ku, int32_t nrhs, int32_t pivoting,
                              int32_t p_hint, double r13, int32_t cap, int32_t *p, int64_t *bounds,
                              int32_t *kinds);

/* ---- factorization ----
 * Stream-ordered: returns once the factorization is enqueued on `stream` (a
 * host band is uploaded first).  Its host-side completion -- the exactly
 * singular pivot check of factorize.cpp:133-257 / kernels.cpp:94-101, boost
 * counts, the coupling paths -- happens at the first call that consumes the
 * factorization (spk_solve, spk_xsolve_begin, spk_fact_*), which reports
 * SPK_ESINGULAR there, or explicitly with spk_fact_sync (what the reference's
 * throwing factorize() maps to). */
spk_status spk_factorize(const double *band, int32_t band_mem, int64_t n, int32_t kl, int32_t ku,
                         const spk_plan *plan, const spk_factor_options *opts, void *stream,
                         spk_fact **out);
/* waits for the factorization and reports its status (SPK_ESINGULAR) */
spk_status spk_fact_sync(const spk_fact *f);
void spk_fact_destroy(spk_fact *f);
/* cudaStreamSynchronize(stream): completes stream-ordered host-memory solves */
spk_status spk_stream_sync(void *stream);

/* ---- multi-GPU slabs (no reference counterpart: the
 * reference is single-node fork-join, parallel_util.hpp:13-45) ----
 * Rows [R_g, R_g + n) of a global system factored on one GPU as its own SPIKE
 * system whose edge partitions also carry the spikes that couple them to the
 * neighbouring slabs; the local reduced hierarchy ends in one unit.
 * band: packed columns [-k*open_left, n + k*open_right) of the slab, k =
 * max(kl, ku) (k halo columns per open edge; device or host). */
spk_status spk_factorize_slab(const double *band, int32_t band_mem, int64_t n, int32_t kl,
                              int32_t ku, const spk_plan *plan, const spk_factor_options *opts,
                              int32_t open_left, int32_t open_right, void *stream,
                              spk_fact **out);
/* Which engine factored f: 0 the general stage programs, 1 the small-k
 * engine (spk_smallk.cu: kl, ku <= 16, non-pivoting), 2 the small-k engine
 * whose reduced hierarchy fell back to the general programs (a pair needed the
 * pivoted 2k coupling); -1 on error.  Waits for the factorization. */
int32_t spk_fact_engine(const spk_fact *f);
/* Debug hook: a device buffer of 2 x 65536 u64 the small-k engine's
 * cooperative kernels stamp with %globaltimer per (level phase, CTA, mark)
 * (factor hierarchy at [0, 65536), forward solve after it); null disables. */
void spk_debug_set_trace(void *d_buf);
/* bit 0: open left edge, bit 1: open right edge */
int32_t spk_fact_open(const spk_fact *f);
/* The slab unit's tips [vt; vb; wt; wb] (4 blocks of k*k column-major, device):
 * top and bottom k rows of its V / W spikes over the slab's reduced rows;
 * zero blocks where the edge is closed.  These are one "partition" of the
 * slab-level reduced system (spk_reduced_create with p = number of slabs). */
spk_status spk_fact_unit_tips(const spk_fact *f, double *d_tips, void *stream);

/* Slab solve with exchange points (device buffers).  Forward: begin exports
 * [y_top; y_bot] (2k x nrhs); the caller solves the slab-level reduced system
 * and steps with [x_top of the right slab; x_bot of the left slab].
 * Transpose: begin exports [chat_0^T tau_t; bhat_last^T tau_b] (2k x nrhs); step
 * 1 imports [left slab's bhat^T tau_b; right slab's chat^T tau_t] and exports
 * [t_top; t_bot; V_int^T t; W_int^T t] (4k x nrhs); step 2 imports [z_top; z_bot]
 * of this slab from the slab-level transposed reduced solve and finishes X.
 * Blocks are column-major with ld = their row count. */
typedef struct spk_xsolve spk_xsolve;
int32_t spk_xsolve_exchanges(const spk_fact *f, int32_t transpose);
spk_status spk_xsolve_begin(const spk_fact *f, int32_t transpose, const double *d_F, int64_t ldf,
                            int32_t nrhs, double *d_X, int64_t ldx, void *stream,
                            double *d_export, spk_xsolve **out);
spk_status spk_xsolve_step(spk_xsolve *x, const double *d_import, double *d_export);
void spk_xsolve_end(spk_xsolve *x);

/* Fields of SpikeFactorization (factorize.hpp:56-74).  Host mirrors copied on
 * demand; these synchronise the factorization's stream. */
spk_status spk_fact_info(const spk_fact *f, int64_t *n, int32_t *kl, int32_t *ku, int32_t *k,
                         int32_t *p, int32_t *levels, int32_t *boost_count,
                         int32_t *boost_warnings);
spk_status spk_fact_bounds(const spk_fact *f, int64_t *bounds /* p+1 */);
spk_status spk_fact_factor_sweeps(const spk_fact *f, int64_t *sweeps /* p */);
spk_status spk_fact_tip(const spk_fact *f, int32_t which, int32_t i, double *out /* k*k */);
/* Level l, unit u spike columns (v: which=0, w: which=1); rows returned in *h.
 * out may be NULL to query h; returns zeros where never formed. */
spk_status spk_fact_level_spike(const spk_fact *f, int32_t l, int32_t which, int32_t u, int32_t *h,
                                double *out);
/* Factored 2k x 2k coupling of level l pair a: packed LU (column-major, 2k x 2k,
 * unit-lower L below the diagonal, U on and above), pivots (0-based rows), and
 * whether the pivoted factorization fell back to boosting. */
spk_status spk_fact_coupling(const spk_fact *f, int32_t l, int32_t a, double *lu, int32_t *piv,
                             int32_t *fell_back);
int32_t spk_fact_units(const spk_fact *f, int32_t l);

/* ---- solves ---- */
typedef struct spk_solve_stats {
    int64_t *partition_full_sweeps; /* p entries or NULL (SolveStats, solve.hpp:11-20) */
    int64_t reduced_coupling_solves;
} spk_solve_stats;

/* X := A^-1 F (transpose=0) or A^-T F (transpose=1); F, X column-major with
 * leading dimensions ldf, ldx >= n.  X may alias F.  mem = SPK_MEM_HOST with
 * nrhs >= 32 (pinned buffers) is pipelined over column chunks and
 * stream-ordered: uploads start at once (under a still running factorization),
 * the call returns without waiting, and X is complete once `stream` is
 * synchronised (spk_stream_sync).  Smaller host solves complete before return. */
spk_status spk_solve(const spk_fact *f, int32_t transpose, const double *F, int64_t ldf,
                     int32_t nrhs, double *X, int64_t ldx, int32_t mem, void *stream,
                     spk_solve_stats *stats);

/* ---- verification and refinement on the device ----
 * All blocks are device pointers (column-major, leading dimensions >= n);
 * only per-column scalars come back to the host. */
/* R = F - op(A) X (band_ops.cpp:11-37 band_matmul, the residual of
 * band_ops.cpp:45-57); d_R may be NULL (not stored).  out (host, 4*ncols):
 * per column c {||r_c||_2^2, ||f_c||_2^2, max|r_c|, max|x_c|}, deterministic. */
spk_status spk_residual_device(const double *d_band, int64_t n, int32_t kl, int32_t ku, const double *d_X,
                               int64_t ldx, const double *d_F, int64_t ldf, int32_t ncols,
                               int32_t transpose, double *d_R, int64_t ldr, void *stream, double *out);
/* out (host, 3): ||A||_1, ||A||_inf, max|a_ij| (band_ops.cpp:59-69 norm1 / max_abs) */
spk_status spk_band_norms_device(const double *d_band, int64_t n, int32_t kl, int32_t ku, void *stream,
                                 double *out);
/* RefineResult (solve.hpp:38-44) without x: X is refined in place */
typedef struct spk_refine_result {
    int32_t iterations;
    int32_t converged;
    int32_t stagnated;
    double residual;
} spk_refine_result;
/* iterative_refine (solve.cpp:404-432, solve.hpp:49-51) on the device: residual
 * r = F - op(A) X on the tensor cores, ||r||_F / ||F||_F to the host, correction
 * solve with the factorization, X += d; stops at tol, at max_iters, or when the
 * residual shrinks by less than 1.1x (stagnated).  band is A, packed
 * ((kl+ku+1) x n); X holds x0 on entry and the refined x on return.  mem:
 * SPK_MEM_DEVICE (all device pointers) or SPK_MEM_HOST (staged; the loop still
 * runs on the device).  Completes before returning. */
spk_status spk_refine(const spk_fact *f, const double *band, const double *F, int64_t ldf, int32_t nrhs,
                      double *X, int64_t ldx, int32_t transpose, int32_t max_iters, double tol, int32_t mem,
                      void *stream, spk_refine_result *res);
/* Hager's 1-norm condition estimate ||A||_1 * est(||A^-1||_1) (oracle.cpp:132-166,
 * condition_estimate_1norm) with the factorization's forward/transpose solves;
 * band on the device or the host (mem). */
spk_status spk_condest_1norm(const spk_fact *f, const double *band, int32_t mem, void *stream, double *cond);

/* ---- .spkb band files (band_io.cpp:98-143 read_spkb / write_matrix; SURVEY.md
 * section 8(f) row 3) ----
 * Format: "SPKB", then n, kl, ku as little-endian int64, then the packed band
 * (kl+ku+1 little-endian doubles per column, columns 0..n-1), i.e. exactly the
 * BandedMatrix / spk_factorize layout.  Errors: SPK_EIO with the reference's
 * messages ("bad SPKB magic", "bad SPKB dimensions", "SPKB file truncated",
 * "cannot open <path>"). */
spk_status spk_spkb_header(const char *path, int64_t *n, int32_t *kl, int32_t *ku);
/* Columns [col0, col0+ncols) of the packed band into dst ((kl+ku+1) x ncols).
 * mem = SPK_MEM_DEVICE streams the file through pinned buffers straight into
 * HBM (file reads overlap the uploads; a slab loads its own column window with
 * its halos); SPK_MEM_HOST reads into host memory.  Completes before return. */
spk_status spk_spkb_load(const char *path, int64_t col0, int64_t ncols, double *dst, int32_t mem,
                         void *stream);
/* Write a packed band (device or host memory) as .spkb. */
spk_status spk_spkb_store(const char *path, const double *band, int64_t n, int32_t kl, int32_t ku,
                          int32_t mem, void *stream);

/* ---- reduced system on its own (reduce_factorize / reduced_solve) ----
 * vt, vb, wt, wb: p blocks of k*k column-major each (host). */
spk_status spk_reduced_create(const double *vt, const double *vb, const double *wt,
                              const double *wb, int32_t p, int32_t k, double boost_eps,
                              spk_reduced **out);
/* The same from device tips: d_tips holds p units of [vt; vb; wt; wb] (4 k x k
 * column-major blocks each, the layout spk_fact_unit_tips writes, e.g. an
 * all-gather of the slabs' unit tips); assembled and factored on `stream`,
 * no host copy of the tips. */
spk_status spk_reduced_create_device(const double *d_tips, int32_t p, int32_t k, double boost_eps,
                                     void *stream, spk_reduced **out);
spk_status spk_reduced_solve(const spk_reduced *r, int32_t transpose, double *z /* host 2pk x ncols */,
                             int32_t ncols, int64_t *couplings);
/* Same on a device block (2pk x ncols, ld 2pk), ordered on stream. */
spk_status spk_reduced_solve_device(const spk_reduced *r, int32_t transpose, double *d_z,
                                    int32_t ncols, void *stream);
int32_t spk_reduced_levels(const spk_reduced *r);
/* The hierarchy's factorization object, for the spk_fact_level_spike /
 * spk_fact_coupling / spk_fact_units getters (owned by r). */
const spk_fact *spk_reduced_fact(const spk_reduced *r);
/* The reduced-system solve of a factorization on its own (2pk tip block). */
spk_status spk_fact_reduced_solve(const spk_fact *f, int32_t transpose, double *z, int32_t ncols,
                                  int64_t *couplings);
/* Test/debug hook: copy the packed LU pool (0), row-major copies (1) or 1/u_jj
 * (2) to out (may be NULL); returns the element count. */
int64_t spk_fact_dump(const spk_fact *f, int32_t which, double *out);
int32_t spk_reduced_boost_warnings(const spk_reduced *r);
void spk_reduced_destroy(spk_reduced *r);

/* ---- device utilities ---- */
/* Y := A X or A^T X with A banded (both on device or both host). */
spk_status spk_band_matmul(const double *band, int64_t n, int32_t kl, int32_t ku, const double *X,
                           int64_t ldx, int32_t ncols, int32_t transpose, double *Y, int64_t ldy,
                           int32_t mem, void *stream);
/* Seeded BASELINE generator (include/spike_b200_gen.h) straight into device
 * memory: band (kl+ku+1) x n column-major; F n x ncols. */
spk_status spk_generate_band(uint64_t seed, int64_t n, int32_t kl, int32_t ku, double dd,
                             double *d_band, void *stream);
spk_status spk_generate_rhs(uint64_t seed, int64_t n, int32_t ncols, double *d_F, int64_t ldf,
                            void *stream);
/* The same global matrix / RHS restricted to a slab: band columns
 * [col0, col0 + ncols) of the n x n system (entries outside the matrix are
 * zero, so halo columns past either end come out empty); F rows
 * [row0, row0 + nrows). */
spk_status spk_generate_band_cols(uint64_t seed, int64_t n, int32_t kl, int32_t ku, double dd,
                                  int64_t col0, int64_t ncols, double *d_band, void *stream);
spk_status spk_generate_rhs_rows(uint64_t seed, int64_t row0, int64_t nrows, int32_t ncols,
                                 double *d_F, int64_t ldf, void *stream);
/* Device arena: freed factor/scratch blocks are cached for reuse by later calls
 * (stream-ordered).  cached = bytes held; trim returns them to the driver. */
int64_t spk_arena_cached(void);
void spk_arena_trim(void);

/* Number of kernel launches issued by this library on the calling thread
 * since the last reset (instrumentation for bench.py's gpu_launches). */
int64_t spk_launch_count(int32_t reset);
/* Of those, launches of the generic correctness-baseline kernels (per-column
 * sweeps, unblocked LU) on SPIKE-partition stages no tuned kernel covers (all
 * generic kernels under spk_set_generic_path).  Zero on the BASELINE
 * configurations; bench.py reports it. */
int64_t spk_generic_launch_count(int32_t reset);
/* Test hook: 1 routes every stage of factorizations created afterwards (and
 * all solves) through the generic kernels, the correctness baseline the tuned
 * kernels are compared against; 0 restores the tuned dispatch.  Process-wide. */
void spk_set_generic_path(int32_t on);

/* Optional per-kernel-class CUDA-event timing (calling thread): launches are
 * bracketed by events on their stream; spk_profile_read drains and returns
 * accumulated device time, algorithmic flops and bytes per class. */
void spk_profile_enable(int32_t on);
int32_t spk_profile_classes(void);
const char *spk_profile_read(int32_t cls, double *ms, double *flops, double *bytes, int64_t *launches);
void spk_profile_reset(void);

/* ---- multi-GPU data plane (spk_dist.cu): one slab of rows per GPU, the
 * reduced-system tip blocks exchanged by NCCL all-gathers; the slab-level
 * reduced system (reduce_factorize, factorize.cpp:46-120, p = number of
 * GPUs) assembled on every GPU from the gathered tips.  No reference
 * counterpart: the reference is single-node (parallel_util.hpp:13-45).
 * NCCL is loaded at run time (libnccl.so.2; SPK_NCCL_LIB overrides); its
 * absence or a collective failure is SPK_ENCCL. */
typedef struct spk_comm spk_comm;
typedef struct spk_dist spk_dist;
#define SPK_COMM_ID_BYTES 128
/* rank 0 creates the id and shares it (any side channel), then every rank
 * initialises; or wrap an existing ncclComm_t (not owned) */
spk_status spk_comm_unique_id(uint8_t *id /* SPK_COMM_ID_BYTES */);
spk_status spk_comm_init(const uint8_t *id, int32_t nranks, int32_t rank, spk_comm **out);
spk_status spk_comm_wrap(void *nccl_comm, int32_t nranks, int32_t rank, spk_comm **out);
void spk_comm_destroy(spk_comm *c);
/* Collective: this rank's slab (d_band: packed columns with k halo columns per
 * open edge, as spk_factorize_slab; edges open toward rank-1 / rank+1) is
 * factored, the unit tips all-gathered, the slab-level system factored. */
spk_status spk_dist_factorize(const double *d_band, int64_t n_local, int32_t kl, int32_t ku,
                              const spk_plan *plan, const spk_factor_options *opts, spk_comm *comm,
                              void *stream, spk_dist **out);
/* Collective: this rank's rows of X := A^-1 F (transpose: A^-T F), device
 * buffers; one (forward) or two (transpose) all-gathers of tip blocks. */
spk_status spk_dist_solve(const spk_dist *d, int32_t transpose, const double *d_F, int64_t ldf,
                          int32_t nrhs, double *d_X, int64_t ldx, void *stream);
const spk_fact *spk_dist_slab(const spk_dist *d);
void spk_dist_destroy(spk_dist *d);
const char *spk_dist_last_error(void);
/* The exchange arithmetic between the all-gathers (distributed.py's
 * formulas), exported for virtual-rank tests: gathered blocks of G ranks ->
 * the slab-level right-hand side / this rank's import. */
enum {
    SPK_XCH_FWD_TOP_RHS = 0, /* (G, nrhs, 2k) -> z (2Gk x nrhs)                        */
    SPK_XCH_FWD_IMPORT = 1,  /* z -> [x_top(rank+1); x_bot(rank-1)] (2k x nrhs)        */
    SPK_XCH_TR_IMPORT1 = 2,  /* (G, nrhs, 2, k) -> [bhat^T tau_b(rank-1); chat^T tau_t(rank+1)] */
    SPK_XCH_TR_TOP_RHS = 3,  /* (G, nrhs, 4, k) -> t - C^T t_int (2Gk x nrhs)          */
    SPK_XCH_TR_IMPORT2 = 4   /* z -> this rank's [z_top; z_bot] (2k x nrhs)            */
};
spk_status spk_dist_exchange(int32_t op, const double *d_src, double *d_dst, int32_t G, int32_t rank,
                             int32_t k, int32_t nrhs, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SPIKE_B200_H */
