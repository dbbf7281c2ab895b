"""The small-k engine (spk_smallk.cu: kl, ku <= 16, non-pivoting; partitions
of <= 384 rows; k_sk_parts / k_sk_levels / k_sk_solve) against the CPU oracle
and against the general engine on the same plan: spike tips, reduced levels,
forward solves on the engine's own kernel (nrhs <= 8) and on the general
programs (wider forward solves, every transpose solve, on the small-k
factors), and the hierarchy fallback for pairs that need the pivoted 2k
coupling (|W| > 1)."""
import numpy as np
import pytest

from conftest import rel_componentwise

pytestmark = pytest.mark.gpu

CASES = [
    # n, kl, ku, p, dd
    (20000, 16, 16, 104, 2.0),
    (6000, 5, 9, 31, 1.5),
    (9001, 9, 3, 47, 1.3),
    (3000, 1, 1, 17, 1.5),
    (12345, 12, 16, 65, 1.2),
    (2000, 16, 16, 6, 1.5),
    (700, 2, 2, 2, 1.5),
]


@pytest.mark.parametrize("n,kl,ku,p,dd", CASES)
@pytest.mark.parametrize("nrhs", [1, 3, 8, 12])
def test_smallk_engine_vs_oracle(oracle, spk, n, kl, ku, p, dd, nrhs):
    band = oracle.generate_band(3100 + n + kl + 7 * ku, n, kl, ku, dd)
    F = np.asfortranarray(oracle.generate_rhs(3200 + n, n, nrhs))
    a = spk.BandedMatrix(n, kl, ku, band)
    plan = spk.gpu_plan(n, kl, ku, nrhs, False, p)
    fact = spk.factorize(a, plan)
    assert spk.fact_engine(fact) == 1
    for tr in (False, True):
        X = spk.transpose_solve(fact, F) if tr else spk.solve(fact, F)
        Xo = oracle.oracle_solve(band, n, kl, ku, F, tr, True)
        res = oracle.relative_residual(band, n, kl, ku, X, F, tr)
        assert res <= 1e-12 and rel_componentwise(X, Xo) <= 1e-10, (tr, res)
    # tips and the reduced hierarchy against the general engine on the same plan
    with spk.generic_path():
        g = spk.factorize(a, plan)
    assert spk.fact_engine(g) == 0
    for w in ("vt", "vb", "wt", "wb", "bhat", "chat"):
        for i in range(plan.p):
            assert rel_componentwise(getattr(fact, w)[i], getattr(g, w)[i]) <= 1e-12, (w, i)
    for l in range(fact.levels.levels()):
        for u in range(len(fact.levels.v[l])):
            assert rel_componentwise(fact.levels.v[l][u], g.levels.v[l][u]) <= 1e-11, (l, u)
            assert rel_componentwise(fact.levels.w[l][u], g.levels.w[l][u]) <= 1e-11, (l, u)
    assert fact.factor_sweeps == g.factor_sweeps and fact.boost_count == g.boost_count
    # bit-deterministic
    assert np.array_equal(spk.solve(spk.factorize(a, plan), F), spk.solve(fact, F))


def test_smallk_boosting_matches_general(oracle, spk):
    """Exact zero first pivots: the engine boosts the same pivots as the
    general LU (kernels.cpp:104-109)."""
    n, k, p = 4000, 8, 21
    band = oracle.generate_band(77, n, k, k, 1.5)
    plan = spk.gpu_plan(n, k, k, 2, False, p)
    for r in [0] + plan.bounds[1:-1] + [n - 1]:
        band[r, k] = 0.0
    a = spk.BandedMatrix(n, k, k, band)
    fact = spk.factorize(a, plan)
    assert spk.fact_engine(fact) in (1, 2)
    with spk.generic_path():
        g = spk.factorize(a, plan)
    assert fact.boost_count == g.boost_count == p
    F = oracle.generate_rhs(78, n, 2)
    assert rel_componentwise(spk.solve(fact, F), spk.solve(g, F)) <= 1e-8


def test_smallk_hierarchy_fallback(oracle, spk):
    """Weakly dominant bands with |W| > 1 in some pairs: the hierarchy falls
    back to the general programs (pivoted 2k couplings); results unchanged."""
    n, k, p = 6000, 4, 40
    band = oracle.generate_band(91, n, k, k, 0.6)
    F = np.asfortranarray(oracle.generate_rhs(92, n, 3))
    a = spk.BandedMatrix(n, k, k, band)
    plan = spk.gpu_plan(n, k, k, 3, False, p)
    fact = spk.factorize(a, plan)
    eng = spk.fact_engine(fact)
    assert eng in (1, 2)
    with spk.generic_path():
        g = spk.factorize(a, plan)
    for tr in (False, True):
        X = spk.transpose_solve(fact, F) if tr else spk.solve(fact, F)
        Xg = spk.transpose_solve(g, F) if tr else spk.solve(g, F)
        assert rel_componentwise(X, Xg) <= 1e-8, (eng, tr)
