"""CPU tests: the C restatement (oracle/spike_oracle.c) pinned to the golden
fixtures produced by the compiled reference (tests/golden/make_golden.py).

These run without a GPU and without /root/reference.
"""
import os

import numpy as np
import pytest

from conftest import rel_componentwise

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
SEED = 20181108
BOOST_TOL = 1e-8


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def cases(g):
    return sorted({k.split("/")[0] for k in g.files if "/" in k and not k.startswith("reduced_")})


def test_golden_file_present(gold):
    assert len(cases(gold)) >= 8


@pytest.mark.parametrize("name", ["c1_small", "c2_small", "c3_small", "c4_small", "asym", "asym_piv",
                                  "dual_mix", "serial", "k1"])
def test_oracle_matches_reference(oracle, gold, name):
    n, kl, ku, nrhs, t, piv = [int(x) for x in gold[name + "/shape"]]
    dd = float(gold[name + "/dd"][0])
    band = oracle.generate_band(SEED, n, kl, ku, dd)
    F = oracle.generate_rhs(SEED + 1, n, nrhs)
    # same inputs as the reference saw
    cs = gold[name + "/band_checksum"]
    assert band.sum() == cs[0] and np.abs(band).sum() == cs[1]
    bounds = [int(b) for b in gold[name + "/bounds"]]
    fact = oracle.factorize(band, n, kl, ku, bounds, bool(piv))
    x, sw, cc = fact.solve(F, False)
    xt, swt, cct = fact.solve(F, True)
    tol = 1e-9 if piv else 1e-12
    assert rel_componentwise(x, gold[name + "/x"]) <= tol
    assert rel_componentwise(xt, gold[name + "/xt"]) <= tol
    assert sw == list(gold[name + "/sweeps"]) and swt == list(gold[name + "/sweeps_t"])
    assert [cc, cct] == list(gold[name + "/couplings"])
    assert fact.factor_sweeps() == list(gold[name + "/factor_sweeps"])
    assert [fact.levels, fact.boost_count] == list(gold[name + "/levels"])
    for w in ("vt", "vb", "wt", "wb", "bhat", "chat"):
        ref = gold[name + "/" + w]
        for i in range(len(bounds) - 1):
            assert rel_componentwise(fact.tip(w, i), ref[i]) <= (1e-9 if piv else 1e-12), (w, i)
    # the reference's own serial banded GE oracle
    xo = oracle.oracle_solve(band, n, kl, ku, F, False, True)
    assert rel_componentwise(xo, gold[name + "/x_oracle_solve"]) <= 1e-13
    rr = oracle.relative_residual(band, n, kl, ku, x, F, False)
    assert rr <= 1e-12


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_reduced_matches_reference(oracle, gold, p, k):
    pre = f"reduced_p{p}_k{k}/"
    tips = [gold[pre + w] for w in ("vt", "vb", "wt", "wb")]
    y = gold[pre + "y"]
    z, c = oracle.reduced_solve_tips(*tips, p, k, y, False)
    zt, ct = oracle.reduced_solve_tips(*tips, p, k, y, True)
    assert rel_componentwise(z, gold[pre + "z"]) <= 1e-13
    assert rel_componentwise(zt, gold[pre + "zt"]) <= 1e-13
    assert [c, ct] == list(gold[pre + "couplings"])


def test_oracle_planner_matches_reference(oracle, gold):
    for row in gold["plans"]:
        n, k, t, nrhs, p, tu, idle = [int(x) for x in row[:7]]
        r12, r13 = oracle.compute_ratios(1.0, nrhs, k)
        pl = oracle.make_plan(n, k, k, t, r12, r13)
        assert pl["p"] == p and pl["threads_used"] == tu and pl["idle_threads"] == idle
        exp = [int(b) for b in row[7:] if b >= 0]
        assert pl["bounds"][:len(exp)] == exp


def test_reference_oracle_cross_check_when_available(oracle, reference):
    """Where oracle/_ref exists (this container), re-run a random case live."""
    if reference is None:
        pytest.skip("oracle/_ref not built here")
    n, k, nrhs = 1500, 5, 3
    band = oracle.generate_band(99, n, k, k, 1.3)
    F = oracle.generate_rhs(100, n, nrhs)
    rf = reference.factorize_t(band, n, k, k, 6, 1.0, 2.0, False)
    of = oracle.factorize(band, n, k, k, rf.bounds(), False)
    for tr in (False, True):
        assert rel_componentwise(rf.solve(F, tr)[0], of.solve(F, tr)[0]) <= 1e-12


def test_oracle_boosted_factorization_matches_reference(oracle, gold):
    """Diagonal boosting (kernels.cpp:104-109): exact zero first pivots in every
    partition.  The restatement boosts the same pivots (count) and its boosted
    solution equals the reference's to rounding."""
    n, kl, ku, nrhs, t, piv = [int(x) for x in gold["boost/shape"]]
    band = gold["boost/band"]
    F = gold["boost/F"]
    bounds = [int(b) for b in gold["boost/bounds"]]
    fact = oracle.factorize(band, n, kl, ku, bounds, False)
    assert fact.boost_count == int(gold["boost/boost_count"][0]) == len(bounds) - 1
    x, _, _ = fact.solve(F, False)
    xt, _, _ = fact.solve(F, True)
    # a boosted pivot is sqrt(eps) max|A_i|: rounding differences between two
    # correct implementations grow by up to 1/sqrt(eps) through it
    assert rel_componentwise(x, gold["boost/x"]) <= BOOST_TOL
    assert rel_componentwise(xt, gold["boost/xt"]) <= BOOST_TOL
    # the reference's refinement converged to the true solution
    xo = oracle.oracle_solve(band, n, kl, ku, F, False, True)
    assert rel_componentwise(gold["boost/x_refined"], xo) <= 1e-12
    assert gold["boost/refine"][0][1] == 1 and gold["boost/refine"][1][1] == 1
