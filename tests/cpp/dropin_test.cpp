// dropin_test.cpp — the reference's C++ API used unchanged against the B200
// library: same calls and checks as the reference suites
// (proj/tests/test_solve_stage.cpp, test_factor_ds.cpp), written here as a
// plain main() (the reference's doctest header is not vendored).
#include "spike/band_io.hpp"
#include "spike/factorize.hpp"
#include "spike/partition.hpp"
#include "spike/solve.hpp"

#include <cmath>
#include <cstdio>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

using namespace spike;

static int failures = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);     \
            ++failures;                                                    \
        }                                                                  \
    } while (0)

static double urand(uint64_t& s) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    return (double)(s >> 11) * (1.0 / 9007199254740992.0);
}

static BandedMatrix make_dd(int n, int kl, int ku, double dd, uint64_t seed) {
    BandedMatrix a(n, kl, ku);
    for (int j = 0; j < n; ++j) {
        double col = 0.0;
        for (int i = std::max(0, j - ku); i <= std::min(n - 1, j + kl); ++i)
            if (i != j) {
                const double v = urand(seed);
                a.set(i, j, v);
                col += v;
            }
        a.set(j, j, dd * col + 1e-3);
    }
    return a;
}

static DenseBlock make_rhs(int n, int c, uint64_t seed) {
    DenseBlock f(n, c);
    for (double& v : f.data) v = urand(seed);
    return f;
}

static double max_abs_diff(const DenseBlock& a, const DenseBlock& b) {
    double m = 0.0;
    for (std::size_t i = 0; i < a.data.size(); ++i) m = std::max(m, std::fabs(a.data[i] - b.data[i]));
    return m;
}

int main() {
    {  // identity returns F exactly (test_solve_stage.cpp:45-53)
        BandedMatrix a(32, 1, 1);
        for (int i = 0; i < 32; ++i) a.set(i, i, 1.0);
        SpikeFactorization fact = factorize(a, make_plan(32, 1, 1, 4, 1.0, 2.0));
        DenseBlock f = make_rhs(32, 2, 3);
        CHECK(max_abs_diff(solve(fact, f), f) == 0.0);
        CHECK(max_abs_diff(transpose_solve(fact, f), f) == 0.0);
    }
    {  // p=2 and p=8-mixed: residual gate (test_solve_stage.cpp:55-80)
        for (int t : {2, 12}) {
            const int n = 4096, k = 8;
            BandedMatrix a = make_dd(n, k, k, 1.5, 11 + t);
            DenseBlock f = make_rhs(n, 4, 13);
            for (bool piv : {false, true}) {
                SpikeFactorization fact = factorize(a, make_plan(n, k, k, t, 1.2, 2.4), {piv, default_boost_eps()});
                DenseBlock x = solve(fact, f);
                CHECK(relative_residual(a, x, f) < 1e-12);
                DenseBlock xt = transpose_solve(fact, f);
                CHECK(relative_residual(a, xt, f, true) < 1e-12);
            }
        }
    }
    {  // non-power-of-two partition counts (extension)
        const int n = 6000, k = 10;
        BandedMatrix a = make_dd(n, k, k, 1.2, 7);
        DenseBlock f = make_rhs(n, 3, 9);
        for (int p : {3, 5, 7, 11}) {
            SpikeFactorization fact = factorize(a, gpu_plan(n, k, k, 3, false, p));
            CHECK(fact.p() == p);
            CHECK(relative_residual(a, solve(fact, f), f) < 1e-12);
            CHECK(relative_residual(a, transpose_solve(fact, f), f, true) < 1e-12);
        }
    }
    {  // sweep budget and coupling count (test_solve_stage.cpp:196-216)
        const int n = 1024, k = 4;
        BandedMatrix a = make_dd(n, k, k, 1.5, 59);
        SpikeFactorization fact = factorize(a, make_plan(n, k, k, 4, 1.0, 2.0));
        SolveStats st;
        solve(fact, make_rhs(n, 2, 61), &st);
        CHECK((st.partition_full_sweeps == std::vector<long>{2, 4, 4, 2}));
        CHECK(st.reduced_coupling_solves == 3);
        CHECK((fact.factor_sweeps == std::vector<long>{0, 3, 3, 0}));
    }
    {  // reduced levels of a factorization solve the assembled reduced system
        const int n = 240, k = 3;
        BandedMatrix a = make_dd(n, k, k, 1.5, 31);
        SpikeFactorization fact = factorize(a, make_plan(n, k, k, 4, 1.0, 2.0));
        const int p = fact.p(), N = 2 * p * k;
        std::vector<double> S((size_t)N * N, 0.0);
        for (int i = 0; i < N; ++i) S[(size_t)i * N + i] = 1.0;
        for (int i = 0; i < p; ++i)
            for (int c = 0; c < k; ++c)
                for (int r = 0; r < k; ++r) {
                    if (i + 1 < p) {
                        S[(size_t)(2 * (i + 1) * k + c) * N + 2 * i * k + r] = fact.vt[i].at(r, c);
                        S[(size_t)(2 * (i + 1) * k + c) * N + (2 * i + 1) * k + r] = fact.vb[i].at(r, c);
                    }
                    if (i > 0) {
                        S[(size_t)((2 * i - 1) * k + c) * N + 2 * i * k + r] = fact.wt[i].at(r, c);
                        S[(size_t)((2 * i - 1) * k + c) * N + (2 * i + 1) * k + r] = fact.wb[i].at(r, c);
                    }
                }
        DenseBlock y = make_rhs(N, 2, 37);
        long cnt = 0;
        DenseBlock x = reduced_solve(fact.levels, y, &cnt);
        CHECK(cnt == p - 1);
        double worst = 0.0;  // residual of S x = y
        for (int c = 0; c < 2; ++c)
            for (int i = 0; i < N; ++i) {
                double s = 0.0;
                for (int j = 0; j < N; ++j) s += S[(size_t)j * N + i] * x.at(j, c);
                worst = std::max(worst, std::fabs(s - y.at(i, c)));
            }
        CHECK(worst < 1e-12);
    }
    {  // error behaviour: shape errors and an exactly singular pivot column
        const int n = 64, k = 2;
        BandedMatrix a = make_dd(n, k, k, 1.5, 107);
        SpikeFactorization fact = factorize(a, make_plan(n, k, k, 4, 1.0, 2.0));
        DenseBlock wrong(n + 1, 1);
        bool threw = false;
        try {
            solve(fact, wrong);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        DenseBlock empty(n, 0);
        CHECK(solve(fact, empty).cols == 0);
        BandedMatrix z(n, k, k);
        for (int i = 0; i < n; ++i) z.set(i, i, 1.0);
        z.set(5, 5, 0.0);
        threw = false;
        try {
            factorize(z, make_plan(n, k, k, 2, 1.0, 2.0), {true, default_boost_eps()});
        } catch (const std::runtime_error&) {
            threw = true;
        }
        CHECK(threw);
    }
    {  // refinement recovers a boosted factorization (test_solve_stage.cpp:246-259)
        const int n = 200, k = 3;
        BandedMatrix a = make_dd(n, k, k, 1.5, 89);
        a.set(0, 0, 0.0);
        SpikeFactorization fact = factorize(a, make_plan(n, k, k, 2, 1.0, 2.0));
        CHECK(fact.boost_count >= 1);
        DenseBlock f = make_rhs(n, 2, 97);
        RefineResult r = iterative_refine(fact, a, f, DenseBlock(n, 2), 5, 1e-12);
        CHECK(r.converged);
        CHECK(relative_residual(a, r.x, f) <= 1e-12);
    }
    {  // band_io.hpp: .spkb round trip through the reference's write_matrix / read_matrix
        const int n = 300, kl = 3, ku = 5;
        BandedMatrix a = make_dd(n, kl, ku, 1.5, 123);
        const std::string path = "dropin_tmp.spkb";
        write_matrix(a, path, MatrixFormat::Spkb);
        BandedMatrix b = read_matrix(path);
        CHECK(b.n() == n && b.kl() == kl && b.ku() == ku && b.data() == a.data());
        bool threw = false;
        try {
            read_matrix(path, 4, 5);
        } catch (const std::runtime_error&) {
            threw = true;
        }
        CHECK(threw);
        std::remove(path.c_str());
    }
    {  // partition.hpp calibration and its cache; oracle.hpp condition estimate
        CalibrationResult c = calibrate_k(20000, 8, 3);
        CHECK(c.k > 0.0 && c.factor_seconds > 0.0 && c.solve_seconds > 0.0);
        const std::string path = "dropin_k.cache";
        write_k_cache(path, c.k);
        CHECK(read_k_cache(path).value_or(-1.0) == c.k);
        std::remove(path.c_str());
        CHECK(!read_k_cache("no_such_k.cache").has_value());
        const int n = 400, k = 3;
        BandedMatrix a = make_dd(n, k, k, 1.2, 131);
        SpikeFactorization fact = factorize(a, gpu_plan(n, k, k, 1, false, 4));
        const double cond = condition_estimate_1norm(fact, a);
        CHECK(cond >= 1.0 && std::isfinite(cond));
    }
    std::printf(failures ? "DROPIN FAIL %d\n" : "DROPIN PASS\n", failures);
    return failures ? 1 : 0;
}
