// spk_launch.h — host-side launch wrappers of the device kernels.
#pragma once

#include <cuda_runtime.h>

#include "spk_device.cuh"

namespace spk {

void count_launch(int n = 1);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel,
// size), thread-safe; a failure raises SPK_ECUDA (spk_capi.cu)
void set_smem_attr(const void* fn, int bytes);
// multiprocessors of the current device (cached per device)
int device_sms();

void launch_fill_factors(const double* band, long long n, int akl, int aku, const PartDev* d_parts,
                         int nparts, long long max_elems, double* fac, int* piv, unsigned long long* amax,
                         cudaStream_t s);
void launch_band_lu(const int* d_units, int nunits, const PartDev* d_parts, double* fac, int* piv,
                    const unsigned long long* amax, double boost_eps, int* boost_cnt,
                    int* fell_back, int* status, const int* flags, cudaStream_t s);
// units with m <= 160 factored in shared memory (spk_kernels_generic.cu);
// false when a unit is larger (caller falls back to launch_band_lu)
bool launch_band_lu_small(const int* d_units, int nunits, int max_m, const PartDev* d_parts, double* fac,
                          int* piv, const unsigned long long* amax, double boost_eps, int* boost_cnt,
                          int* fell_back, int* status, const int* flags, cudaStream_t s,
                          bool redo_only = false);
// short units staged in shared memory (spk_kernels_generic.cu); false when
// the shape is not covered (caller falls back to launch_sweep)
bool launch_sweep_small(const SweepJob* d_jobs, int njobs, int max_nc, int chunks, int maxr,
                        const PartDev* d_parts, const double* fac, const int* piv, const Bufs& B, int ncols,
                        cudaStream_t s);
void launch_sweep(const SweepJob* d_jobs, int njobs, int max_nc, const PartDev* d_parts,
                  const double* fac, const int* piv, const Bufs& B, int ncols, cudaStream_t s);
void launch_copy(const CopyJob* d_jobs, int njobs, long long max_elems, const Bufs& B, int ncols,
                 cudaStream_t s);
void launch_gemm(const GemmJob* d_jobs, int njobs, int max_r, int max_nc, const Bufs& B, int ncols,
                 cudaStream_t s);
void launch_gemm_dmma(const GemmJob* d_jobs, int njobs, int max_r, int max_nc, const Bufs& B, int ncols,
                      cudaStream_t s, double* ws = nullptr, int nsplit = 1);
int gemm_splitk_factor(int njobs, int max_r, int max_nc, int max_kk);
size_t gemm_splitk_workspace(int njobs, int max_r, int max_nc, int nsplit);
void launch_copy_cols(const double* src, long long lds, double* dst, long long ldd, long long n, int ncols,
                      cudaStream_t s);
void launch_corners(const double* band, long long n, int akl, int aku, const long long* d_bounds,
                    int p, int k, int open_l, int open_r, double* bhat, double* chat, cudaStream_t s);
void launch_build_coupling(const CouplingJob* d_jobs, int njobs, long long max_elems,
                           const PartDev* d_parts, const double* pool, double* fac, int* piv,
                           unsigned long long* amax, const int* flags, cudaStream_t s);
void launch_wcheck(const CouplingJob* d_jobs, int njobs, int k, const double* pool, int* flags, cudaStream_t s);
void launch_schur_init(const CouplingJob* d_jobs, int njobs, long long max_elems, const PartDev* d_parts,
                       double* fac, int* piv, const int* flags, cudaStream_t s);
bool launch_schur_inverse(const CouplingJob* d_jobs, int njobs, int n, const PartDev* d_parts, const double* fac,
                          double* pool, int* flags, cudaStream_t s);
void launch_dense_lu(const CouplingJob* d_jobs, int njobs, int n, const PartDev* d_parts, double* fac, int* piv,
                     int* flags, cudaStream_t s);
// spk_verify.cu: verification and refinement kernels
void launch_band_mm(const double* band, long long n, int kl, int ku, const double* X, long long ldx, int ncols,
                    int transpose, const double* F, long long ldf, double* Y, long long ldy, cudaStream_t s);
int col_stats_blocks(long long n);
void launch_col_stats(const double* X, long long ldx, long long n, int ncols, double* part, double* out,
                      cudaStream_t s);
void launch_band_norms(const double* band, long long n, int kl, int ku, unsigned long long* out, cudaStream_t s);
void launch_axpy(double* X, long long ldx, const double* D, long long ldd, long long n, int ncols, cudaStream_t s);
void launch_sign(const double* y, double* xi, long long n, cudaStream_t s);
int dot_argmax_blocks(long long n);
void launch_dot_argmax(const double* z, const double* x, long long n, double* part, cudaStream_t s);
void launch_unit(double* x, long long n, long long j, cudaStream_t s);
void launch_fill(double* x, long long n, double v, cudaStream_t s);
void launch_band_matmul(const double* band, long long n, int kl, int ku, const double* X,
                        long long ldx, int ncols, int transpose, double* Y, long long ldy,
                        cudaStream_t s);
struct FastSweepArgs;
bool launch_sweep_fast_fl(int tr, int nc, bool piv, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A,
                          cudaStream_t s);
bool launch_sweep_fast_bu(int tr, int nc, bool piv, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A,
                          cudaStream_t s);
bool launch_sweep_fast_fut(int tr, int nc, bool piv, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A,
                           cudaStream_t s);
bool launch_sweep_fast_blt(int tr, int nc, bool piv, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A,
                           cudaStream_t s);
// non-pivoting blocked DMMA band LU (spk_lu_fast.cu)
struct FastLuArgs {
    const int* units;
    const PartDev* parts;
    const double* band;  // input band (kl+ku+1) x n, column-major; column 0 of the partitions' rows
    int akl, aku;
    double* fac;
    double* tfac;  // row-major copy, or null (made on demand)
    double* dinv;
    int* piv;
    double boost_eps;
    int* boost_cnt;
    // readable band columns around `band` (TMA staging of the entering
    // blocks): columns [-col0, ncols - col0); ncols = 0 disables TMA
    long long ncols;
    long long col0;
};
bool launch_band_lu_fast(const int* d_units, int nunits, int kmax, const FastLuArgs& A, cudaStream_t s);
// blocked pivoted band LU on the tensor cores (spk_lu_piv_dmma.cu); false
// when the band is wider than its tile windows (kl+ku > 192)
struct PivDmmaArgs {
    const int* units;
    const PartDev* parts;
    const double* band;
    int akl, aku;
    double* fac;
    double* tfac;  // row-major copy (row i: (i, i-kl .. i+ubw) at [kl + c - i])
    double* dinv;  // 1 / u_jj
    int* piv;
    int* status;
    double* lblk;  // blocked L records (spk_piv_blocked.cuh), or null
    // dense coupling units (launch_dense_lu_piv_dmma): factored in place from
    // the band layout in `fac` (its backup on the fallback), job guards, and
    // the per-unit redo marker (2) for an exactly singular unit
    const int* flags;
    int* redo;
};
bool launch_band_lu_piv_dmma(int nunits, int kl, int ku, const PivDmmaArgs& A, cudaStream_t s);
// the pivoted 2k x 2k coupling units (m <= 128) on the same kernel; false when
// not covered.  Units marked for redo need k_band_lu_small (its fallback).
bool launch_dense_lu_piv_dmma(int nunits, int max_m, const PivDmmaArgs& A, cudaStream_t s);
// blocked pivoted forward L sweep from the LU's records (spk_sweep_piv_dmma.cu)
struct PivSweepArgs {
    const SweepJob* jobs;
    const PartDev* parts;
    const double* lblk;
    Bufs B;
    int ncols;
    // the transposed sweep's unaligned first panel runs the reference's
    // per-row steps from the packed gbtf2 factor and pivots
    const double* fac;
    const int* piv;
};
bool launch_sweep_piv_dmma(int trw, int nwarps, dim3 grid, const PivSweepArgs& A, cudaStream_t s);
// pivoted transposed L sweep (B := P^T L^-T B) from the same records
bool launch_sweep_piv_dmma_t(int trw, int nwarps, dim3 grid, const PivSweepArgs& A, cudaStream_t s);
struct PivLuArgs;
bool launch_band_lu_piv(const int* d_units, int nunits, int kl, int ku, const PivLuArgs& A, cudaStream_t s);
bool launch_sweep_dmma2_fl(int ntw, int ncw, dim3 grid, const FastSweepArgs& A, cudaStream_t s,
                           bool pair = false);
bool launch_sweep_dmma2_bu(int ntw, int ncw, dim3 grid, const FastSweepArgs& A, cudaStream_t s,
                           bool pair = false);
bool launch_sweep_dmma2_fut(int ntw, int ncw, dim3 grid, const FastSweepArgs& A, cudaStream_t s,
                           bool pair = false);
bool launch_sweep_dmma2_blt(int ntw, int ncw, dim3 grid, const FastSweepArgs& A, cudaStream_t s,
                           bool pair = false);
bool launch_sweep_dmma_fl(int ntw, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A, cudaStream_t s,
                          bool pair = false);
bool launch_sweep_dmma_bu(int ntw, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A, cudaStream_t s,
                          bool pair = false);
bool launch_sweep_dmma_fut(int ntw, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A, cudaStream_t s,
                          bool pair = false);
bool launch_sweep_dmma_blt(int ntw, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A, cudaStream_t s,
                          bool pair = false);
void launch_transpose_factors(const PartDev* d_parts, int nparts, long long max_elems, const double* fac,
                              double* tfac, double* dinv, cudaStream_t s);

// ---------------------------------------------------------------------------
// small-k engine (spk_smallk.cu): non-pivoting bands with kl, ku <= 31.  One
// warp per partition for the partition work (register-window LU, spike tips),
// one cooperative persistent kernel for the reduced hierarchy and one for the
// forward solve, levels separated by a grid barrier.
struct SkUnit {
    long long voff, woff;  // pool offsets of the unit's V / W spike (h x k, ld h), -1: none
    int uh, uoff;          // height (rows of the reduced system), first reduced row
};
struct SkPair {
    long long sinv;            // pool offset of S^-1 (k x k, ld k)
    long long vl, wl, vr, wr;  // pool offsets of the children's spikes (left / right unit), -1: none
    long long nv, nw;          // the merged unit's spikes, -1: none
    int hL, hR;                // children heights
    int zb;                    // first reduced row of the merged unit
    int gidx;                  // flag index (1 = Schur path)
    int left;                  // global index of the left unit (right = left + 1)
    int next;                  // global index of the merged unit on the next level
};
struct SkItem {
    int pair;  // >= 0: pair (global index); < 0: carried unit -(pair + 1) (global unit index)
    int row0;  // first row of this item's chunk of the merged unit
    int next;  // carried unit: its global index on the next level
    int pad;
};
struct SkLevel {
    int item0, nitems;     // row items (pairs' merged units, the carried unit)
    int pair0, npairs;     // pairs of the level (global indices)
    int carry, carry_next; // carried odd unit (global index on this / the next level), -1: none
};
constexpr int kSkChunk = 128;  // merged-unit rows per work item
struct SkPartsArgs {
    const double* band;
    long long n;
    int akl, aku, k, p;
    const PartDev* parts;
    double* fac;   // packed LU (the row-major copy follows lazily, ensure_tfac)
    double* dinv;
    int* boost;
    double* pool;
    long long off_bhat, off_chat;
    const SkUnit* units;  // level 0: one per partition
    double boost_eps;
    int mmax;  // longest partition
};
struct SkLevelsArgs {
    double* pool;
    const SkUnit* units;
    const SkPair* pairs;
    const SkItem* items;
    const SkLevel* levels;
    int nlevels, k;
    int* flags;
    double boost_eps;  // an exactly singular Schur complement: its zero pivots boosted
    unsigned* bar;     // grid barrier: {count, generation}, zeroed
    unsigned long long* trace;  // debug: globaltimer per (phase, CTA, mark), or null
};
struct SkSolveArgs {
    const PartDev* parts;
    int p, k, nrhs;
    const double* fac;
    long long fac_size;  // doubles in the factor pool (bulk copies stay inside it)
    const double* pool;
    long long off_bhat, off_chat;
    const SkUnit* units;
    const SkPair* pairs;
    const SkItem* items;
    const SkLevel* levels;
    int nlevels;
    const double* F;
    long long ldf;
    double* X;
    long long ldx;
    double* T;  // reduced right-hand sides (2pk x nrhs, ld 2pk), updated in place
    double* ZS;     // per pair: z2 and z1 (2 x 16 x NR, row-major), for the deferred row updates
    unsigned* cnt;  // per-pair arrival counters of the reduced-solve tree, zeroed
    unsigned* bar;
    int mmax, rmax;  // longest partition, largest packed column height
    unsigned long long* trace;  // debug: globaltimer per (phase, CTA, mark), or null
};
// debug hook (spk_debug_set_trace): device buffer the small-k kernels stamp
extern unsigned long long* g_sk_trace;
// false when the shape is not covered (kl or ku > 31)
bool launch_sk_parts(const SkPartsArgs& A, cudaStream_t s);
void launch_sk_levels(const SkLevelsArgs& A, cudaStream_t s);
// forward solve, nrhs <= kSkMaxRhs; its dynamic shared memory (the caller
// checks it fits)
constexpr int kSkMaxRhs = 8;
size_t sk_solve_smem(int mmax, int rmax, int nrhs);
void launch_sk_solve(const SkSolveArgs& A, cudaStream_t s);

void launch_generate_band(unsigned long long seed, long long n, int kl, int ku, double dd, long long col0,
                          long long ncols, double* band, cudaStream_t s);
void launch_generate_rhs(unsigned long long seed, long long row0, long long nrows, int ncols, double* F,
                         long long ldf, cudaStream_t s);

}  // namespace spk
