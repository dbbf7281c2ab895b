"""K calibration and the ratio sweep on the GPU."""
import numpy as np
import pytest

from conftest import rel_componentwise

pytestmark = pytest.mark.gpu


def test_calibrate_k(spk):
    r = spk.calibrate_k(40000, 8, 3)
    assert r.k > 0 and r.factor_seconds > 0 and r.solve_seconds > 0
    r0 = spk.calibrate_k(0, 4, 1)  # n_sample <= 0 -> 200 k
    assert r0.k > 0 and r0.timer_warning  # far below the 10 ms clock threshold
    with pytest.raises(spk.InvalidArgument):
        spk.calibrate_k(100, 0, 1)


@pytest.mark.parametrize("r13", [0.5, 1.7])
def test_ratio_plan_solves_like_oracle(oracle, spk, r13):
    n, k, nrhs = 12000, 6, 3
    band = oracle.generate_band(31, n, k, k, 1.4)
    F = np.asfortranarray(oracle.generate_rhs(32, n, nrhs))
    a = spk.BandedMatrix(n, k, k, band)
    plan = spk.gpu_plan(n, k, k, nrhs, False, 7, r13=r13)
    fact = spk.factorize(a, plan)
    for tr in (False, True):
        X = spk.transpose_solve(fact, F) if tr else spk.solve(fact, F)
        xo = oracle.oracle_solve(band, n, k, k, F, tr, True)
        assert rel_componentwise(X, xo) <= 1e-10
        assert oracle.relative_residual(band, n, k, k, X, F, tr) <= 1e-12


def test_sweep_ratios(spk, tmp_path, monkeypatch):
    from paper_1811_03559_b200 import tuning

    monkeypatch.setenv("SPIKE_K_CACHE", str(tmp_path / "k.cache"))
    spk.write_k_cache(tmp_path / "k.cache", 1.0)
    grid = tuning.sweep_ratios(60000, 8, 4, [0.75, 1.0, 1.5], p=12, reps=2)
    assert len(grid) == 4 and grid[-1].calculated and not any(g.calculated for g in grid[:-1])
    r12, r13 = spk.compute_ratios(1.0, 4, 8)
    assert (grid[-1].r12, grid[-1].r13) == (r12, r13)
    assert all(g.factor_seconds > 0 and g.solve_seconds > 0 for g in grid)
    csv = tuning.format_csv(grid)
    assert csv.splitlines()[0] == "r12,r13,factor_seconds,solve_seconds,total_seconds,flag"
    assert csv.splitlines()[-1].startswith("# gain_from_best_measured: factor=")
