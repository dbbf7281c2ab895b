// ref_shim.cpp — C entry points over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles the
// reference sources in place (/root/reference/proj/src/*.cpp, read-only) plus
// this file into oracle/_ref/libspike_ref.so.  It is used (a) to generate the
// golden fixtures under tests/golden/ that pin oracle/spike_oracle.c, and
// (b) by bench.py --impl reference / cpu_baseline to time the reference's own
// CPU path (spike::make_plan -> factorize -> solve / transpose_solve).
#include "spike/band_io.hpp"
#include "spike/band_ops.hpp"
#include "spike/factorize.hpp"
#include "spike/oracle.hpp"
#include "spike/partition.hpp"
#include "spike/solve.hpp"

#include "../include/spike_b200_gen.h"

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

using namespace spike;

namespace {
thread_local std::string g_err;

BandedMatrix band_from(const double* band, int n, int kl, int ku) {
    BandedMatrix a(n, kl, ku);
    std::memcpy(a.data().data(), band, sizeof(double) * a.data().size());
    return a;
}

DenseBlock block_from(const double* x, int rows, int cols) {
    DenseBlock b(rows, cols);
    if (rows * static_cast<std::size_t>(cols))
        std::memcpy(b.data.data(), x, sizeof(double) * b.data.size());
    return b;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

struct RefHandle {
    BandedMatrix a;
    SpikeFactorization fact;
};
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_hw_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

void ref_compute_ratios(double K, int nrhs, int k, double* r12, double* r13) {
    auto [a, b] = compute_ratios(K, nrhs, k);
    *r12 = a;
    *r13 = b;
}

// bounds: p+1 ints, kinds: p ints (0 FirstLast, 1 InnerSingle, 2 InnerDual); cap >= p
int ref_make_plan(int n, int kl, int ku, int t, double r12, double r13, int cap, int* p,
                  int* bounds, int* kinds, int* threads_used, int* idle) {
    return guarded([&] {
        PartitionPlan pl = make_plan(n, kl, ku, t, r12, r13);
        *p = pl.p;
        *threads_used = pl.threads_used;
        *idle = pl.idle_threads;
        for (int i = 0; i <= pl.p && i <= cap; ++i) bounds[i] = pl.bounds[i];
        for (int i = 0; i < pl.p && i < cap; ++i) kinds[i] = static_cast<int>(pl.kinds[i]);
    });
}

void* ref_factorize(const double* band, int n, int kl, int ku, int t, double r12, double r13,
                    int pivoting) {
    RefHandle* h = nullptr;
    const int rc = guarded([&] {
        auto* hh = new RefHandle{band_from(band, n, kl, ku), {}};
        PartitionPlan pl = make_plan(n, kl, ku, t, r12, r13);
        hh->fact = factorize(hh->a, pl, {pivoting != 0, default_boost_eps()});
        h = hh;
    });
    return rc == 0 ? h : nullptr;
}

// Factorize with an explicit (power-of-two) plan given as bounds; all inner
// partitions single-thread.
void* ref_factorize_bounds(const double* band, int n, int kl, int ku, int p, const int* bounds,
                           int pivoting) {
    RefHandle* h = nullptr;
    const int rc = guarded([&] {
        auto* hh = new RefHandle{band_from(band, n, kl, ku), {}};
        PartitionPlan pl;
        pl.p = p;
        pl.bounds.assign(bounds, bounds + p + 1);
        pl.kinds.assign(p, PartitionKind::InnerSingle);
        pl.kinds.front() = PartitionKind::FirstLast;
        pl.kinds.back() = PartitionKind::FirstLast;
        pl.threads_used = p;
        hh->fact = factorize(hh->a, pl, {pivoting != 0, default_boost_eps()});
        h = hh;
    });
    return rc == 0 ? h : nullptr;
}

void ref_free(void* h) { delete static_cast<RefHandle*>(h); }

int ref_fact_p(void* h) { return static_cast<RefHandle*>(h)->fact.p(); }
int ref_fact_boost_count(void* h) { return static_cast<RefHandle*>(h)->fact.boost_count; }
int ref_fact_levels(void* h) { return static_cast<RefHandle*>(h)->fact.levels.levels(); }
void ref_fact_factor_sweeps(void* h, long* out) {
    const auto& f = static_cast<RefHandle*>(h)->fact;
    for (int i = 0; i < f.p(); ++i) out[i] = f.factor_sweeps[i];
}
void ref_fact_bounds(void* h, int* out) {
    const auto& f = static_cast<RefHandle*>(h)->fact;
    for (int i = 0; i <= f.p(); ++i) out[i] = f.plan.bounds[i];
}

// which: 0 vt, 1 vb, 2 wt, 3 wb, 4 bhat, 5 chat (k*k, column-major)
void ref_fact_tip(void* h, int which, int i, double* out) {
    const auto& f = static_cast<RefHandle*>(h)->fact;
    const std::vector<DenseBlock>* src[6] = {&f.vt, &f.vb, &f.wt, &f.wb, &f.bhat, &f.chat};
    const DenseBlock& b = (*src[which])[i];
    const std::size_t kk = static_cast<std::size_t>(f.k) * f.k;
    if (b.data.size() == kk) std::memcpy(out, b.data.data(), sizeof(double) * kk);
    else std::memset(out, 0, sizeof(double) * kk);
}

int ref_solve(void* h, const double* F, int nrhs, int transpose, double* X, long* psweeps,
              long* couplings) {
    return guarded([&] {
        const auto& f = static_cast<RefHandle*>(h)->fact;
        DenseBlock fb = block_from(F, f.n, nrhs);
        SolveStats st;
        DenseBlock x = transpose ? transpose_solve(f, fb, &st) : solve(f, fb, &st);
        if (!x.data.empty()) std::memcpy(X, x.data.data(), sizeof(double) * x.data.size());
        if (psweeps)
            for (int i = 0; i < f.p(); ++i) psweeps[i] = st.partition_full_sweeps[i];
        if (couplings) *couplings = st.reduced_coupling_solves;
    });
}

int ref_reduced_solve_tips(const double* vt, const double* vb, const double* wt,
                           const double* wb, int p, int k, double* z, int ncols, int transpose,
                           long* couplings) {
    return guarded([&] {
        const std::size_t kk = static_cast<std::size_t>(k) * k;
        std::vector<DenseBlock> VT(p), VB(p), WT(p), WB(p);
        for (int i = 0; i < p; ++i) {
            VT[i] = block_from(vt + i * kk, k, k);
            VB[i] = block_from(vb + i * kk, k, k);
            WT[i] = block_from(wt + i * kk, k, k);
            WB[i] = block_from(wb + i * kk, k, k);
        }
        ReducedLevels rl = reduce_factorize(VT, VB, WT, WB, p, k);
        DenseBlock y = block_from(z, 2 * p * k, ncols);
        long c = 0;
        DenseBlock x = transpose ? reduced_solve_transpose(rl, y, &c) : reduced_solve(rl, y, &c);
        std::memcpy(z, x.data.data(), sizeof(double) * x.data.size());
        if (couplings) *couplings = c;
    });
}

int ref_oracle_solve(const double* band, int n, int kl, int ku, const double* F, int nrhs,
                     int transpose, int pivoting, double* X) {
    return guarded([&] {
        DenseBlock x = oracle_solve(band_from(band, n, kl, ku), block_from(F, n, nrhs),
                                    transpose != 0, pivoting != 0);
        std::memcpy(X, x.data.data(), sizeof(double) * x.data.size());
    });
}

double ref_condition_estimate_1norm(const double* band, int n, int kl, int ku) {
    double out = -1.0;
    guarded([&] { out = condition_estimate_1norm(band_from(band, n, kl, ku)); });
    return out;
}

double ref_relative_residual(const double* band, int n, int kl, int ku, const double* X,
                             const double* F, int ncols, int transpose) {
    double out = -1.0;
    guarded([&] {
        out = relative_residual(band_from(band, n, kl, ku), block_from(X, n, ncols),
                                block_from(F, n, ncols), transpose != 0);
    });
    return out;
}

// Timed reference CPU path (spike_cli.cpp:119-169 protocol without the CSV):
// make_plan(t) -> factorize -> solve [-> transpose_solve], seconds per stage.
int ref_time_path(const double* band, int n, int kl, int ku, const double* F, int nrhs, int t,
                  double K, int pivoting, int do_transpose, double* t_factor, double* t_solve,
                  double* t_tsolve, double* X, double* XT, int* p_out) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        BandedMatrix a = band_from(band, n, kl, ku);
        DenseBlock fb = block_from(F, n, nrhs);
        auto [r12, r13] = compute_ratios(K, nrhs, std::max(1, std::max(kl, ku)));
        PartitionPlan pl = make_plan(n, kl, ku, t, r12, r13);
        *p_out = pl.p;
        auto t0 = clk::now();
        SpikeFactorization fact = factorize(a, pl, {pivoting != 0, default_boost_eps()});
        auto t1 = clk::now();
        DenseBlock x = solve(fact, fb);
        auto t2 = clk::now();
        *t_factor = std::chrono::duration<double>(t1 - t0).count();
        *t_solve = std::chrono::duration<double>(t2 - t1).count();
        if (X) std::memcpy(X, x.data.data(), sizeof(double) * x.data.size());
        *t_tsolve = 0.0;
        if (do_transpose) {
            auto t3 = clk::now();
            DenseBlock xt = transpose_solve(fact, fb);
            *t_tsolve = std::chrono::duration<double>(clk::now() - t3).count();
            if (XT) std::memcpy(XT, xt.data.data(), sizeof(double) * xt.data.size());
        }
    });
}

// iterative_refine (solve.cpp:404-432) on a reference factorization: X holds
// x0 on entry and the refined x on return; info = {iterations, converged,
// stagnated}
int ref_iterative_refine(void* h, const double* F, int nrhs, double* X, int max_iters, double tol,
                         int transpose, int* info, double* residual) {
    return guarded([&] {
        auto* hh = static_cast<RefHandle*>(h);
        const auto& f = hh->fact;
        RefineResult r = iterative_refine(f, hh->a, block_from(F, f.n, nrhs), block_from(X, f.n, nrhs),
                                          max_iters, tol, transpose != 0);
        if (!r.x.data.empty()) std::memcpy(X, r.x.data.data(), sizeof(double) * r.x.data.size());
        info[0] = r.iterations;
        info[1] = r.converged ? 1 : 0;
        info[2] = r.stagnated ? 1 : 0;
        *residual = r.residual;
    });
}

// band_io.cpp: the reference's own .spkb writer / reader (golden fixtures)
int ref_write_spkb(const double* band, int n, int kl, int ku, const char* path) {
    return guarded([&] { write_matrix(band_from(band, n, kl, ku), path, MatrixFormat::Spkb); });
}

int ref_read_spkb(const char* path, int* n, int* kl, int* ku, double* out) {
    return guarded([&] {
        BandedMatrix a = read_matrix(path);
        *n = a.n();
        *kl = a.kl();
        *ku = a.ku();
        if (out) std::memcpy(out, a.data().data(), sizeof(double) * a.data().size());
    });
}

} // extern "C"
