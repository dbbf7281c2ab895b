// spike_api.cpp — the reference's C++ API (namespace spike) over the C-ABI.
//
// Host-only glue: argument checks and exception types as in the reference
// (SURVEY.md 8(b)), C-ABI calls for everything numerical, and host mirrors of
// the factorization fields the reference's tests introspect.
#include "../../include/spike/spike_b200.hpp"

#include "../../include/spike_b200.h"

#include <algorithm>
#include <cstring>
#include <string>

namespace spike {

namespace {

[[noreturn]] void rethrow(spk_status st) {
    const std::string msg = spk_last_error();
    switch (st) {
        case SPK_EINVAL: throw std::invalid_argument(msg);
        case SPK_EDOMAIN: throw std::domain_error(msg);
        case SPK_ERANGE: throw std::out_of_range(msg);
        case SPK_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

void check(spk_status st) {
    if (st != SPK_OK) rethrow(st);
}

std::vector<int32_t> kinds_of(const PartitionPlan& plan) {
    std::vector<int32_t> k(plan.p, SPK_INNER_SINGLE);
    for (int i = 0; i < plan.p && i < (int)plan.kinds.size(); ++i) k[i] = static_cast<int32_t>(plan.kinds[i]);
    return k;
}

DenseBlock fetch_tip(spk_fact* f, int which, int i, int k) {
    DenseBlock b(k, k);
    check(spk_fact_tip(f, which, i, b.data.data()));
    return b;
}

}  // namespace

// ------------------------------------------------------------------ storage
BandedMatrix::BandedMatrix(int n, int kl, int ku) : n_(n), kl_(kl), ku_(ku) {
    if (n < 1) throw std::invalid_argument("BandedMatrix: n must be >= 1");
    if (kl < 0 || ku < 0 || kl >= n || ku >= n) throw std::invalid_argument("BandedMatrix: need 0 <= kl,ku < n");
    data_.assign(static_cast<std::size_t>(ld()) * n, 0.0);
}

BandedMatrix BandedMatrix::identity(int n) {
    BandedMatrix a(n, 0, 0);
    std::fill(a.data_.begin(), a.data_.end(), 1.0);
    return a;
}

bool BandedMatrix::in_band(int i, int j) const {
    return i >= 0 && j >= 0 && i < n_ && j < n_ && i - j <= kl_ && j - i <= ku_;
}

double BandedMatrix::at(int i, int j) const {
    if (i < 0 || j < 0 || i >= n_ || j >= n_) throw std::out_of_range("BandedMatrix::at: index out of range");
    return in_band(i, j) ? data_[static_cast<std::size_t>(j) * ld() + ku_ + i - j] : 0.0;
}

void BandedMatrix::set(int i, int j, double v) {
    if (!in_band(i, j)) throw std::out_of_range("BandedMatrix::set: entry outside the band");
    data_[static_cast<std::size_t>(j) * ld() + ku_ + i - j] = v;
}

DenseBlock::DenseBlock(int r, int c) : rows(r), cols(c) {
    if (r < 0 || c < 0) throw std::invalid_argument("DenseBlock: negative shape");
    data.assign(static_cast<std::size_t>(r) * c, 0.0);
}
MatView DenseBlock::view() { return {data.data(), rows, cols, rows}; }
ConstMatView DenseBlock::view() const { return {data.data(), rows, cols, rows}; }
MatView DenseBlock::block(int row0, int nrows) { return view().block(row0, nrows); }
ConstMatView DenseBlock::block(int row0, int nrows) const { return view().block(row0, nrows); }

// band_corner (spike2x2.hpp:12, spike2x2.cpp:17-26): the rows x cols block of
// A at (row0, col0), zero where the band (or the matrix) does not reach; the
// B-hat / C-hat corners the device computes in k_corners
DenseBlock band_corner(const BandedMatrix& a, int row0, int col0, int rows, int cols) {
    DenseBlock out(rows, cols);
    for (int j = 0; j < cols; ++j)
        for (int i = 0; i < rows; ++i) {
            const int gi = row0 + i, gj = col0 + j;
            if (a.in_band(gi, gj)) out.at(i, j) = a.at(gi, gj);
        }
    return out;
}

DenseBlock copy_of(ConstMatView v) {
    DenseBlock out(v.rows, v.cols);
    assign(out.view(), v);
    return out;
}
void assign(MatView dst, ConstMatView src) {
    for (int j = 0; j < src.cols; ++j) std::memcpy(dst.col(j), src.col(j), sizeof(double) * src.rows);
}
void subtract_inplace(MatView dst, ConstMatView src) {
    for (int j = 0; j < src.cols; ++j)
        for (int i = 0; i < src.rows; ++i) dst.at(i, j) -= src.at(i, j);
}
void reverse_rows_inplace(MatView v) {
    for (int j = 0; j < v.cols; ++j) std::reverse(v.col(j), v.col(j) + v.rows);
}
DenseBlock reversed_rows(ConstMatView v) {
    DenseBlock out = copy_of(v);
    reverse_rows_inplace(out.view());
    return out;
}
void gemm_minus(MatView c, ConstMatView a, ConstMatView b) {
    for (int j = 0; j < c.cols; ++j)
        for (int l = 0; l < a.cols; ++l) {
            const double s = b.at(l, j);
            for (int i = 0; i < c.rows; ++i) c.at(i, j) -= s * a.at(i, l);
        }
}
void gemm_minus_t(MatView c, ConstMatView a, ConstMatView b) {
    for (int j = 0; j < c.cols; ++j)
        for (int i = 0; i < c.rows; ++i) {
            double s = 0.0;
            for (int l = 0; l < a.rows; ++l) s += a.at(l, i) * b.at(l, j);
            c.at(i, j) -= s;
        }
}

// ------------------------------------------------------------------ planning
int PartitionPlan::dual_count() const {
    return static_cast<int>(std::count(kinds.begin(), kinds.end(), PartitionKind::InnerDual));
}
int PartitionPlan::single_count() const { return p - dual_count(); }

PartitionPlan distribute_threads(int t, int cap_p) {
    const int cap = std::max(2, 2 * t + 2);
    std::vector<int32_t> kinds(cap);
    int32_t p = 0, used = 0, idle = 0;
    check(spk_distribute_threads(t, cap_p, &p, kinds.data(), cap, &used, &idle));
    PartitionPlan plan;
    plan.p = p;
    for (int i = 0; i < p; ++i) plan.kinds.push_back(static_cast<PartitionKind>(kinds[i]));
    plan.threads_used = used;
    plan.idle_threads = idle;
    return plan;
}

std::pair<double, double> compute_ratios(double k_const, int n_rhs, int k) {
    if (k_const <= 0.0) throw std::invalid_argument("compute_ratios: K must be > 0");
    if (k < 1) throw std::invalid_argument("compute_ratios: k must be >= 1");
    if (n_rhs < 0) throw std::invalid_argument("compute_ratios: n_rhs must be >= 0");
    double r12 = 0, r13 = 0;
    spk_compute_ratios(k_const, n_rhs, k, &r12, &r13);
    return {r12, r13};
}

std::vector<int> compute_sizes(int n, const PartitionPlan& skel, double r12, double r13, int min_single,
                               int min_dual) {
    std::vector<int32_t> kinds = kinds_of(skel);
    std::vector<int64_t> sizes(skel.p);
    check(spk_compute_sizes(n, skel.p, kinds.data(), r12, r13, min_single, min_dual, sizes.data()));
    return std::vector<int>(sizes.begin(), sizes.end());
}

static PartitionPlan plan_from(int32_t p, const std::vector<int64_t>& b, const std::vector<int32_t>& k) {
    PartitionPlan plan;
    plan.p = p;
    plan.bounds.assign(b.begin(), b.begin() + p + 1);
    for (int i = 0; i < p; ++i) plan.kinds.push_back(static_cast<PartitionKind>(k[i]));
    return plan;
}

PartitionPlan make_plan(int n, int kl, int ku, int t, double r12, double r13) {
    const int cap = std::max(2, 2 * t + 2);
    std::vector<int64_t> b(cap + 1);
    std::vector<int32_t> k(cap);
    int32_t p = 0, used = 0, idle = 0;
    check(spk_make_plan(n, kl, ku, t, r12, r13, cap, &p, b.data(), k.data(), &used, &idle));
    PartitionPlan plan = plan_from(p, b, k);
    plan.threads_used = used;
    plan.idle_threads = idle;
    plan.r12 = r12;
    plan.r13 = r13;
    return plan;
}

PartitionPlan gpu_plan(int n, int kl, int ku, int nrhs, bool pivoting, int p_hint) {
    const int cap = std::max(4096, 2 * p_hint + 2);
    std::vector<int64_t> b(cap + 1);
    std::vector<int32_t> k(cap);
    int32_t p = 0;
    check(spk_gpu_plan(n, kl, ku, nrhs, pivoting ? 1 : 0, p_hint, cap, &p, b.data(), k.data()));
    PartitionPlan plan = plan_from(p, b, k);
    plan.threads_used = p;
    return plan;
}

// ------------------------------------------------------------------ factors
static void mirror_levels(ReducedLevels& rl, const spk_fact* h, int nlev, int k);

SpikeFactorization factorize(const BandedMatrix& a, const PartitionPlan& plan, FactorOptions opts) {
    if (plan.n() != a.n()) throw std::invalid_argument("factorize: plan does not match matrix");
    for (int i = 0; i < plan.p; ++i)
        if (plan.size(i) < 1) throw std::invalid_argument("factorize: empty partition");
    std::vector<int64_t> bounds(plan.bounds.begin(), plan.bounds.end());
    std::vector<int32_t> kinds = kinds_of(plan);
    spk_plan sp{plan.p, bounds.data(), kinds.data()};
    spk_factor_options so{opts.pivoting ? 1 : 0, opts.boost_eps};
    spk_fact* h = nullptr;
    check(spk_factorize(a.data().data(), SPK_MEM_HOST, a.n(), a.kl(), a.ku(), &sp, &so, nullptr, &h));
    SpikeFactorization f;
    f.handle = std::shared_ptr<void>(h, [](void* q) { spk_fact_destroy(static_cast<spk_fact*>(q)); });
    f.plan = plan;
    f.n = a.n();
    f.kl = a.kl();
    f.ku = a.ku();
    f.k = std::max(a.kl(), a.ku());
    f.options = opts;
    int32_t nlev = 0, boost = 0, warn = 0;
    check(spk_fact_info(h, nullptr, nullptr, nullptr, nullptr, nullptr, &nlev, &boost, &warn));
    f.boost_count = boost;
    std::vector<int64_t> sw(plan.p);
    check(spk_fact_factor_sweeps(h, sw.data()));
    f.factor_sweeps.assign(sw.begin(), sw.end());
    std::vector<DenseBlock>* dst[6] = {&f.vt, &f.vb, &f.wt, &f.wb, &f.bhat, &f.chat};
    for (int w = 0; w < 6; ++w)
        for (int i = 0; i < plan.p; ++i) dst[w]->push_back(fetch_tip(h, w, i, f.k));
    ReducedLevels& rl = f.levels;
    rl.p = plan.p;
    rl.k = f.k;
    rl.boost_warnings = warn;
    rl.device = f.handle;
    mirror_levels(rl, h, nlev, f.k);
    return f;
}

// Host mirrors of the reduced hierarchy (ReducedLevels, factorize.hpp:26-49):
// per level the units' V / W spike columns and the factored 2k coupling blocks
static void mirror_levels(ReducedLevels& rl, const spk_fact* h, int nlev, int k) {
    for (int l = 0; l < nlev; ++l) {
        const int units = spk_fact_units(h, l);
        rl.v.emplace_back();
        rl.w.emplace_back();
        for (int u = 0; u < units; ++u)
            for (int which = 0; which < 2; ++which) {
                int32_t hh = 0;
                check(spk_fact_level_spike(h, l, which, u, &hh, nullptr));
                DenseBlock b(hh, k);
                check(spk_fact_level_spike(h, l, which, u, &hh, b.data.data()));
                (which == 0 ? rl.v : rl.w).back().push_back(std::move(b));
            }
        rl.pairs.emplace_back();
        const int nn = 2 * k;
        for (int a2 = 0; a2 < units / 2; ++a2) {
            std::vector<double> lu(static_cast<std::size_t>(nn) * nn);
            std::vector<int> piv(nn);
            int32_t fb = 0;
            check(spk_fact_coupling(h, l, a2, lu.data(), reinterpret_cast<int32_t*>(piv.data()), &fb));
            rl.pairs.back().emplace_back(nn, std::move(lu), std::move(piv), fb == 0);
        }
    }
}

ReducedLevels reduce_factorize(const std::vector<DenseBlock>& vt, const std::vector<DenseBlock>& vb,
                               const std::vector<DenseBlock>& wt, const std::vector<DenseBlock>& wb, int p, int k,
                               double boost_eps, int) {
    if (p < 1) throw std::invalid_argument("reduce_factorize: p must be >= 1");
    const std::size_t kk = static_cast<std::size_t>(k) * k;
    std::vector<double> packed[4];
    const std::vector<DenseBlock>* src[4] = {&vt, &vb, &wt, &wb};
    for (int w = 0; w < 4; ++w) {
        packed[w].assign(kk * p + 1, 0.0);
        for (int i = 0; i < p && i < (int)src[w]->size(); ++i)
            if ((*src[w])[i].data.size() == kk) std::memcpy(&packed[w][kk * i], (*src[w])[i].data.data(), kk * 8);
    }
    spk_reduced* r = nullptr;
    check(spk_reduced_create(packed[0].data(), packed[1].data(), packed[2].data(), packed[3].data(), p, k,
                             boost_eps, &r));
    ReducedLevels rl;
    rl.p = p;
    rl.k = k;
    rl.standalone = true;
    rl.device = std::shared_ptr<void>(r, [](void* q) { spk_reduced_destroy(static_cast<spk_reduced*>(q)); });
    rl.boost_warnings = spk_reduced_boost_warnings(r);
    if (k > 0) mirror_levels(rl, spk_reduced_fact(r), spk_reduced_levels(r), k);
    return rl;
}

// ------------------------------------------------------------------ solves
static DenseBlock solve_impl(const SpikeFactorization& fact, const DenseBlock& f, SolveStats* stats,
                             bool transpose) {
    if (f.rows != fact.n)
        throw std::invalid_argument(transpose ? "transpose_solve: F.rows must equal n" : "solve: F.rows must equal n");
    DenseBlock x(fact.n, f.cols);
    std::vector<int64_t> sw(fact.p());
    spk_solve_stats st{sw.data(), 0};
    check(spk_solve(static_cast<spk_fact*>(fact.handle.get()), transpose ? 1 : 0, f.data.data(), fact.n, f.cols,
                    x.data.data(), fact.n, SPK_MEM_HOST, nullptr, &st));
    if (stats) {
        stats->partition_full_sweeps.assign(sw.begin(), sw.end());
        stats->reduced_coupling_solves = st.reduced_coupling_solves;
    }
    return x;
}

DenseBlock solve(const SpikeFactorization& fact, const DenseBlock& f, SolveStats* stats) {
    return solve_impl(fact, f, stats, false);
}
DenseBlock transpose_solve(const SpikeFactorization& fact, const DenseBlock& f, SolveStats* stats) {
    return solve_impl(fact, f, stats, true);
}

// ------------------------------------------------------------------ 2x2 kernel
// spike2x2.cpp:246-289 (the standalone wrappers) over a p = 2 factorization
Spike2x2Factors factor_2x2(const BandedMatrix& a, bool pivoting, double boost_eps) {
    const int n = a.n(), k = std::max(a.kl(), a.ku());
    // spike2x2.cpp:37-38
    if (n < 2 * (a.kl() + a.ku() + 1)) throw std::invalid_argument("Spike2x2Factors: partition too small for its band");
    Spike2x2Factors fac;
    fac.n_ = n;
    fac.k_ = k;
    fac.split_ = (n + 1) / 2;
    PartitionPlan plan;
    plan.p = 2;
    plan.bounds = {0, fac.split_, n};
    plan.kinds = {PartitionKind::FirstLast, PartitionKind::FirstLast};
    plan.threads_used = 2;
    FactorOptions opts;
    opts.pivoting = pivoting;
    opts.boost_eps = boost_eps;
    fac.fact_ = factorize(a, plan, opts);
    if (k > 0) {
        fac.vtip_ = fac.fact_.vb[0];
        fac.wtip_ = fac.fact_.wt[1];
        if (!fac.fact_.levels.pairs.empty() && !fac.fact_.levels.pairs[0].empty())
            fac.reduced_ = fac.fact_.levels.pairs[0][0];
    }
    return fac;
}

DenseBlock solve_2x2(const Spike2x2Factors& fac, const DenseBlock& f, bool transpose, SweepCounter* counter) {
    DenseBlock x = transpose ? transpose_solve(fac.factorization(), f) : solve(fac.factorization(), f);
    // two half-sweep pairs per solve (spike2x2.hpp:36-41)
    if (counter) counter->full_sweeps_solve += 2;
    return x;
}

SpikeTips spikes_2x2(const Spike2x2Factors& fac, const DenseBlock& bhat, const DenseBlock& chat,
                     SweepCounter* counter) {
    const int n = fac.n(), k = fac.k();
    if (bhat.rows != k || bhat.cols != k || chat.rows != k || chat.cols != k)
        throw std::invalid_argument("spikes_2x2: corner blocks must be k x k");
    SpikeTips t;
    t.vt = DenseBlock(k, k);
    t.vb = DenseBlock(k, k);
    t.wt = DenseBlock(k, k);
    t.wb = DenseBlock(k, k);
    if (k > 0) {
        // one solve with the 2k columns [0; bhat] and [chat; 0]
        DenseBlock rhs(n, 2 * k);
        for (int c = 0; c < k; ++c)
            for (int i = 0; i < k; ++i) {
                rhs.at(n - k + i, c) = bhat.at(i, c);
                rhs.at(i, k + c) = chat.at(i, c);
            }
        const DenseBlock x = solve(fac.factorization(), rhs);
        for (int c = 0; c < k; ++c)
            for (int i = 0; i < k; ++i) {
                t.vt.at(i, c) = x.at(i, c);
                t.vb.at(i, c) = x.at(n - k + i, c);
                t.wt.at(i, c) = x.at(i, k + c);
                t.wb.at(i, c) = x.at(n - k + i, k + c);
            }
    }
    // three half-sweep pairs for spike generation (spike2x2.hpp:46-48)
    if (counter) counter->full_sweeps_factor += 3;
    return t;
}

static DenseBlock reduced_impl(const ReducedLevels& levels, const DenseBlock& y, long* couplings, bool transpose) {
    if (y.rows != 2 * levels.p * levels.k)
        throw std::invalid_argument(transpose ? "reduced_solve_transpose: tip block has wrong height"
                                              : "reduced_solve: tip block has wrong height");
    DenseBlock z = y;
    int64_t c = 0;
    if (levels.standalone) {
        check(spk_reduced_solve(static_cast<spk_reduced*>(levels.device.get()), transpose ? 1 : 0, z.data.data(),
                                z.cols, &c));
    } else {
        check(spk_fact_reduced_solve(static_cast<spk_fact*>(levels.device.get()), transpose ? 1 : 0, z.data.data(),
                                     z.cols, &c));
    }
    if (couplings) *couplings += c;
    return z;
}

DenseBlock reduced_solve(const ReducedLevels& levels, const DenseBlock& y, long* couplings, int) {
    return reduced_impl(levels, y, couplings, false);
}
DenseBlock reduced_solve_transpose(const ReducedLevels& levels, const DenseBlock& g, long* couplings, int) {
    return reduced_impl(levels, g, couplings, true);
}

// ------------------------------------------------------------------ band ops
DenseBlock band_matmul(const BandedMatrix& a, const DenseBlock& x, bool transpose) {
    if (x.rows != a.n()) throw std::invalid_argument("band_matmul: X.rows must equal n");
    DenseBlock y(a.n(), x.cols);
    if (x.cols)
        check(spk_band_matmul(a.data().data(), a.n(), a.kl(), a.ku(), x.data.data(), a.n(), x.cols,
                              transpose ? 1 : 0, y.data.data(), a.n(), SPK_MEM_HOST, nullptr));
    return y;
}

double frobenius_norm(const DenseBlock& b) {
    double s = 0.0;
    for (double v : b.data) s += v * v;
    return std::sqrt(s);
}

double relative_residual(const BandedMatrix& a, const DenseBlock& x, const DenseBlock& f, bool transpose) {
    if (x.rows != a.n() || f.rows != a.n() || x.cols != f.cols)
        throw std::invalid_argument("relative_residual: inconsistent shapes");
    const double fn = frobenius_norm(f);
    if (fn == 0.0) {
        if (frobenius_norm(x) == 0.0) return 0.0;
        throw std::domain_error("relative_residual: F is zero but X is not");
    }
    DenseBlock r = band_matmul(a, x, transpose);
    for (std::size_t i = 0; i < r.data.size(); ++i) r.data[i] -= f.data[i];
    return frobenius_norm(r) / fn;
}

double norm1(const BandedMatrix& a) {
    double best = 0.0;
    for (int j = 0; j < a.n(); ++j) {
        double s = 0.0;
        for (int q = 0; q < a.ld(); ++q) s += std::fabs(a.col(j)[q]);
        best = std::max(best, s);
    }
    return best;
}

double max_abs(const BandedMatrix& a) {
    double best = 0.0;
    for (double v : a.data()) best = std::max(best, std::fabs(v));
    return best;
}

// A^T as a band: packed column j of A^T holds row j of A (kl and ku swap)
BandedMatrix band_transpose(const BandedMatrix& a) {
    BandedMatrix t(a.n(), a.ku(), a.kl());
    for (int i = 0; i < a.n(); ++i)
        for (int j = std::max(0, i - a.kl()); j <= std::min(a.n() - 1, i + a.ku()); ++j) t.set(j, i, a.at(i, j));
    return t;
}

// solve.cpp:404-432, the loop on the device (spk_refine): residual on the
// tensor cores, correction solves, only ||r||_F / ||F||_F per iteration to the host
RefineResult iterative_refine(const SpikeFactorization& fact, const BandedMatrix& a, const DenseBlock& f,
                              const DenseBlock& x0, int max_iters, double tol, bool transpose) {
    if (f.rows != a.n() || x0.rows != f.rows || x0.cols != f.cols)
        throw std::invalid_argument("iterative_refine: F.rows must equal n");
    RefineResult res;
    res.x = x0;
    spk_refine_result r{};
    check(spk_refine(static_cast<spk_fact*>(fact.handle.get()), a.data().data(), f.data.data(), f.rows, f.cols, res.x.data.data(), res.x.rows,
                     transpose ? 1 : 0, max_iters, tol, SPK_MEM_HOST, nullptr, &r));
    res.iterations = r.iterations;
    res.residual = r.residual;
    res.converged = r.converged != 0;
    res.stagnated = r.stagnated != 0;
    return res;
}

double condition_estimate_1norm(const SpikeFactorization& fact, const BandedMatrix& a) {
    double c = 0.0;
    check(spk_condest_1norm(static_cast<spk_fact*>(fact.handle.get()), a.data().data(), SPK_MEM_HOST, nullptr, &c));
    return c;
}

void write_matrix(const BandedMatrix& a, const std::string& path, MatrixFormat fmt) {
    if (fmt != MatrixFormat::Spkb) throw std::runtime_error("write_matrix: only the SPKB format is supported");
    check(spk_spkb_store(path.c_str(), a.data().data(), a.n(), a.kl(), a.ku(), SPK_MEM_HOST, nullptr));
}

BandedMatrix read_matrix(const std::string& path, std::optional<int> expected_kl, std::optional<int> expected_ku) {
    int64_t n = 0;
    int32_t kl = 0, ku = 0;
    check(spk_spkb_header(path.c_str(), &n, &kl, &ku));
    if ((expected_kl && *expected_kl != kl) || (expected_ku && *expected_ku != ku))
        throw std::runtime_error("SPKB bandwidths differ from the expected ones");
    BandedMatrix a(static_cast<int>(n), kl, ku);
    check(spk_spkb_load(path.c_str(), 0, n, a.data().data(), SPK_MEM_HOST, nullptr));
    return a;
}

CalibrationResult calibrate_k(int n_sample, int k_sample, int reps) {
    spk_calibration c{};
    check(spk_calibrate_k(n_sample, k_sample, reps, nullptr, &c));
    return CalibrationResult{c.k, c.factor_seconds, c.solve_seconds, c.timer_warning != 0};
}

std::string default_k_cache_path() {
    char buf[4096];
    check(spk_default_k_cache_path(buf, sizeof buf));
    return buf;
}

void write_k_cache(const std::string& path, double k) { check(spk_write_k_cache(path.c_str(), k)); }

std::optional<double> read_k_cache(const std::string& path) {
    double k = 0.0;
    int32_t found = 0;
    check(spk_read_k_cache(path.c_str(), &k, &found));
    return found ? std::optional<double>(k) : std::nullopt;
}

}  // namespace spike
