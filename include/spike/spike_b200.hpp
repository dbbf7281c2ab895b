// spike_b200.hpp — drop-in C++ API of the B200 SPIKE solver.
//
// Same names, signatures and exception types as the reference artifact's
// headers (proj/include/spike/{banded_matrix,partition,factorize,solve}.hpp),
// implemented over the C-ABI of include/spike_b200.h (libspike_b200.so).  A
// user of the reference switches by including this header (or the forwarding
// headers next to it, which carry the reference's file names) and linking
// libspike_b200.so instead of libspike.a.  The factorization lives in HBM;
// SpikeFactorization keeps an opaque handle plus the host mirrors the
// reference exposes (plan, corner blocks, spike tips, reduced levels, sweep
// counts, boost count).
//
// Differences, all extensions: factorize() accepts any partition count p >= 1
// (the reference requires a power of two inside reduce_factorize), and
// gpu_plan() chooses p for the device.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <utility>
#include <optional>
#include <string>
#include <vector>

namespace spike {

// ---------------------------------------------------------------- storage
// Band-packed square matrix: entry (i,j), -ku <= i-j <= kl, at packed row
// ku+i-j of column j; kl+ku+1 rows, column-major (banded_matrix.hpp:14-67).
class BandedMatrix {
public:
    BandedMatrix() = default;
    BandedMatrix(int n, int kl, int ku);
    static BandedMatrix identity(int n);

    int n() const { return n_; }
    int kl() const { return kl_; }
    int ku() const { return ku_; }
    int ld() const { return kl_ + ku_ + 1; }
    bool in_band(int i, int j) const;
    double at(int i, int j) const;
    void set(int i, int j, double v);
    double* col(int j) { return data_.data() + static_cast<std::size_t>(j) * ld(); }
    const double* col(int j) const { return data_.data() + static_cast<std::size_t>(j) * ld(); }
    std::vector<double>& data() { return data_; }
    const std::vector<double>& data() const { return data_; }

private:
    int n_ = 0, kl_ = 0, ku_ = 0;
    std::vector<double> data_;
};

struct MatView;
struct ConstMatView;

// Column-major dense block (banded_matrix.hpp:73-91).
struct DenseBlock {
    int rows = 0, cols = 0;
    std::vector<double> data;
    DenseBlock() = default;
    DenseBlock(int r, int c);
    double& at(int i, int j) { return data[static_cast<std::size_t>(j) * rows + i]; }
    double at(int i, int j) const { return data[static_cast<std::size_t>(j) * rows + i]; }
    double* col(int j) { return data.data() + static_cast<std::size_t>(j) * rows; }
    const double* col(int j) const { return data.data() + static_cast<std::size_t>(j) * rows; }
    MatView view();
    ConstMatView view() const;
    MatView block(int row0, int nrows);
    ConstMatView block(int row0, int nrows) const;
};

struct MatView {
    double* p = nullptr;
    int rows = 0, cols = 0, ld = 0;
    double& at(int i, int j) const { return p[static_cast<std::size_t>(j) * ld + i]; }
    double* col(int j) const { return p + static_cast<std::size_t>(j) * ld; }
    MatView block(int row0, int nrows) const { return {p + row0, nrows, cols, ld}; }
};

struct ConstMatView {
    const double* p = nullptr;
    int rows = 0, cols = 0, ld = 0;
    ConstMatView() = default;
    ConstMatView(const MatView& v) : p(v.p), rows(v.rows), cols(v.cols), ld(v.ld) {}
    ConstMatView(const double* q, int r, int c, int l) : p(q), rows(r), cols(c), ld(l) {}
    double at(int i, int j) const { return p[static_cast<std::size_t>(j) * ld + i]; }
    const double* col(int j) const { return p + static_cast<std::size_t>(j) * ld; }
    ConstMatView block(int row0, int nrows) const { return {p + row0, nrows, cols, ld}; }
};

DenseBlock copy_of(ConstMatView v);
void assign(MatView dst, ConstMatView src);
void subtract_inplace(MatView dst, ConstMatView src);
void reverse_rows_inplace(MatView v);
DenseBlock reversed_rows(ConstMatView v);
void gemm_minus(MatView c, ConstMatView a, ConstMatView b);
void gemm_minus_t(MatView c, ConstMatView a, ConstMatView b);
// spike2x2.hpp:12: the rows x cols block of A at (row0, col0); zero where the
// band does not reach (the corner blocks B-hat / C-hat)
DenseBlock band_corner(const BandedMatrix& a, int row0, int col0, int rows, int cols);

// ---------------------------------------------------------------- planning
enum class PartitionKind { FirstLast, InnerSingle, InnerDual };

struct PartitionPlan {
    int p = 1;
    std::vector<int> bounds;
    std::vector<PartitionKind> kinds;
    int threads_used = 1;
    int idle_threads = 0;
    double r12 = 1.0, r13 = 2.0;
    int n() const { return bounds.empty() ? 0 : bounds.back(); }
    int size(int i) const { return bounds[i + 1] - bounds[i]; }
    int dual_count() const;
    int single_count() const;
};

PartitionPlan distribute_threads(int t, int cap_p = 0);
std::pair<double, double> compute_ratios(double k_const, int n_rhs, int k);
std::vector<int> compute_sizes(int n, const PartitionPlan& skeleton, double r12, double r13,
                               int min_single, int min_dual);
PartitionPlan make_plan(int n, int kl, int ku, int t, double r12, double r13);
// B200 planner (extension): equal partitions, p chosen for the device (any p).
PartitionPlan gpu_plan(int n, int kl, int ku, int nrhs = 1, bool pivoting = false, int p = 0);

// ---------------------------------------------------------------- factors
inline double default_boost_eps() { return std::sqrt(std::numeric_limits<double>::epsilon()); }

struct FactorOptions {
    bool pivoting = false;
    double boost_eps = default_boost_eps();
};

struct SweepCounter {
    long full_sweeps_factor = 0;
    long full_sweeps_solve = 0;
};

// Read-only view of one factored 2k coupling block (the reference keeps a
// full LUFactors there; tests use uval / lval / pivoting).
class LUFactors {
public:
    LUFactors() = default;
    LUFactors(int n, std::vector<double> dense_lu, std::vector<int> piv, bool pivoting)
        : n_(n), lu_(std::move(dense_lu)), piv_(std::move(piv)), pivoting_(pivoting) {}
    int n() const { return n_; }
    bool pivoting() const { return pivoting_; }
    const std::vector<int>& pivots() const { return piv_; }
    double uval(int i, int j) const { return i <= j ? lu_[static_cast<std::size_t>(j) * n_ + i] : 0.0; }
    double lval(int i, int j) const {
        return i == j ? 1.0 : (i > j ? lu_[static_cast<std::size_t>(j) * n_ + i] : 0.0);
    }

private:
    int n_ = 0;
    std::vector<double> lu_;
    std::vector<int> piv_;
    bool pivoting_ = true;
};

struct ReducedLevels {
    int p = 1, k = 0;
    std::vector<std::vector<DenseBlock>> v, w;
    std::vector<std::vector<LUFactors>> pairs;
    int boost_warnings = 0;
    int levels() const { return static_cast<int>(pairs.size()); }
    int unit_rows(int level) const { return (2 * k) << level; }
    std::shared_ptr<void> device;  // the device hierarchy (spk_reduced / spk_fact)
    bool standalone = false;
};

ReducedLevels reduce_factorize(const std::vector<DenseBlock>& vt, const std::vector<DenseBlock>& vb,
                               const std::vector<DenseBlock>& wt, const std::vector<DenseBlock>& wb, int p,
                               int k, double boost_eps = default_boost_eps(), int threads = 1);

struct SpikeFactorization {
    PartitionPlan plan;
    int n = 0, kl = 0, ku = 0, k = 0;
    FactorOptions options;
    std::vector<DenseBlock> bhat, chat;
    std::vector<DenseBlock> vt, vb, wt, wb;
    ReducedLevels levels;
    std::vector<long> factor_sweeps;
    int boost_count = 0;
    std::shared_ptr<void> handle;  // spk_fact* (HBM-resident factors)

    int p() const { return plan.p; }
    bool is_dual(int i) const { return plan.kinds[i] == PartitionKind::InnerDual; }
};

SpikeFactorization factorize(const BandedMatrix& a, const PartitionPlan& plan, FactorOptions opts = {});

// ---------------------------------------------------------------- solves
struct SolveStats {
    std::vector<long> partition_full_sweeps;
    long reduced_coupling_solves = 0;
    long total_full_sweeps() const {
        long s = 0;
        for (long v : partition_full_sweeps) s += v;
        return s;
    }
};

DenseBlock solve(const SpikeFactorization& fact, const DenseBlock& f, SolveStats* stats = nullptr);
DenseBlock transpose_solve(const SpikeFactorization& fact, const DenseBlock& f, SolveStats* stats = nullptr);
DenseBlock reduced_solve(const ReducedLevels& levels, const DenseBlock& ytips, long* coupling_solves = nullptr,
                         int threads = 1);
DenseBlock reduced_solve_transpose(const ReducedLevels& levels, const DenseBlock& gtips,
                                   long* coupling_solves = nullptr, int threads = 1);

struct RefineResult {
    DenseBlock x;
    int iterations = 0;
    double residual = 0.0;
    bool converged = false;
    bool stagnated = false;
};

RefineResult iterative_refine(const SpikeFactorization& fact, const BandedMatrix& a, const DenseBlock& f,
                              const DenseBlock& x0, int max_iters, double tol, bool transpose = false);

// ---------------------------------------------------------------- spike2x2.hpp
// The two-partition SPIKE kernel (spike2x2.hpp:25-87, spike2x2.cpp:28-289):
// LU on the top half, UL on the bottom half (split at ceil(n/2)), one factored
// 2k coupling block [[I, vtip], [wtip, I]].  On the GPU the two cooperating
// host threads of the reference are the two partitions of a p = 2
// factorization: both halves are factored by the same launch (one CTA each,
// the bottom half on the reversed view), their interface tips meet in the
// coupling unit, and the std::barrier points are the kernel boundaries of the
// stage program.  The *_task entry points (a CPU threading protocol) have no
// GPU counterpart; the standalone wrappers below keep their signatures,
// results, sweep budgets and exceptions.
struct SpikeTips {
    DenseBlock vt, vb, wt, wb;
};

class Spike2x2Factors {
public:
    Spike2x2Factors() = default;
    int n() const { return n_; }
    int k() const { return k_; }
    int split() const { return split_; }
    int boost_count() const { return fact_.boost_count; }
    // bottom tip of A1^-1 [0; Bint] and top tip of A2^-1 [Cint; 0]
    const DenseBlock& vtip() const { return vtip_; }
    const DenseBlock& wtip() const { return wtip_; }
    const LUFactors& reduced() const { return reduced_; }
    // the HBM-resident p = 2 factorization behind it (extension)
    const SpikeFactorization& factorization() const { return fact_; }

private:
    friend Spike2x2Factors factor_2x2(const BandedMatrix&, bool, double);
    int n_ = 0, k_ = 0, split_ = 0;
    DenseBlock vtip_, wtip_;
    LUFactors reduced_;
    SpikeFactorization fact_;
};

Spike2x2Factors factor_2x2(const BandedMatrix& a, bool pivoting, double boost_eps = default_boost_eps());
DenseBlock solve_2x2(const Spike2x2Factors& fac, const DenseBlock& f, bool transpose = false,
                     SweepCounter* counter = nullptr);
// tips of V = A^-1 [0; bhat] and W = A^-1 [chat; 0] (the enclosing partition's spikes)
SpikeTips spikes_2x2(const Spike2x2Factors& fac, const DenseBlock& bhat, const DenseBlock& chat,
                     SweepCounter* counter = nullptr);

// ---------------------------------------------------------------- band ops
DenseBlock band_matmul(const BandedMatrix& a, const DenseBlock& x, bool transpose = false);
double relative_residual(const BandedMatrix& a, const DenseBlock& x, const DenseBlock& f, bool transpose = false);
double frobenius_norm(const DenseBlock& b);
double norm1(const BandedMatrix& a);
double max_abs(const BandedMatrix& a);
// A^T as a band (kl and ku swap), band_ops.hpp
BandedMatrix band_transpose(const BandedMatrix& a);
// Hager's kappa_1 estimate (oracle.hpp condition_estimate_1norm) computed with
// the factorization's GPU solves instead of a serial banded GE
double condition_estimate_1norm(const SpikeFactorization& fact, const BandedMatrix& a);

// ---------------------------------------------------------------- band_io.hpp
// .spkb binary files (band_io.cpp:98-143); MatrixMarket text is not supported
// by the GPU library and throws std::runtime_error.
enum class MatrixFormat { MatrixMarket, Spkb };
void write_matrix(const BandedMatrix& a, const std::string& path, MatrixFormat fmt);
BandedMatrix read_matrix(const std::string& path, std::optional<int> expected_kl = std::nullopt,
                         std::optional<int> expected_ku = std::nullopt);

// ---------------------------------------------------------------- K calibration (partition.hpp:58-74)
struct CalibrationResult {
    double k = 1.0;
    double factor_seconds = 0.0;
    double solve_seconds = 0.0;
    bool timer_warning = false;
};
// timed on the GPU: one partition's factorization and its two-sweep solve
CalibrationResult calibrate_k(int n_sample, int k_sample, int reps = 5);
std::string default_k_cache_path();
void write_k_cache(const std::string& path, double k);
std::optional<double> read_k_cache(const std::string& path);

}  // namespace spike
