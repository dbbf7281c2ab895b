"""K-cache format and the ratio planner's host logic (partition.cpp:149-170;
no GPU needed)."""
import pytest


def test_k_cache_round_trip_and_format(spk, tmp_path):
    p = tmp_path / "k.cache"
    spk.write_k_cache(p, 1.2345678901234567)
    assert p.read_text() == "K 1.2345678901234567\n"  # os.precision(17); "K " << k << "\n"
    assert spk.read_k_cache(p) == 1.2345678901234567
    p.write_text("X 3\nK 2.5\nK 7\n")
    assert spk.read_k_cache(p) == 2.5  # the first K wins
    p.write_text("X 3\n")
    assert spk.read_k_cache(p) is None
    assert spk.read_k_cache(tmp_path / "missing") is None


def test_default_k_cache_path(spk, monkeypatch):
    monkeypatch.delenv("SPIKE_K_CACHE", raising=False)
    assert spk.default_k_cache_path() == "spike_k.cache"
    monkeypatch.setenv("SPIKE_K_CACHE", "/tmp/somewhere/k.cache")
    assert spk.default_k_cache_path() == "/tmp/somewhere/k.cache"


@pytest.mark.parametrize("n,k,p,r13", [(100000, 16, 10, 1.5), (100000, 16, 10, 0.5), (5000, 4, 3, 2.0),
                                       (5000, 4, 2, 3.0), (1000, 2, 1, 1.0)])
def test_gpu_plan_ratio_sizes(spk, n, k, p, r13):
    plan = spk.gpu_plan(n, k, k, 1, False, p, r13=r13)
    b = plan.bounds
    assert plan.p == p and b[0] == 0 and b[-1] == n
    sizes = [b[i + 1] - b[i] for i in range(p)]
    assert all(s >= 2 * k + 1 for s in sizes)
    if p >= 3:
        inner = sizes[1:-1]
        assert max(inner) - min(inner) <= 1
        assert sizes[0] == sizes[-1]
        assert abs(sizes[0] / (sum(inner) / len(inner)) - r13) <= 0.01 * r13 + 2.0 / min(inner)
    with pytest.raises(spk.DomainError):
        spk.gpu_plan(n, k, k, 1, False, p, r13=0.0)
