"""CPU tests of the host side of the product library (no GPU needed):
planning functions against the reference's known answers
(/root/reference/proj/tests/test_partition.cpp), the Python mirror's argument
checking, and the C-ABI surface (every symbol include/spike_b200.h declares is
exported by libspike_b200.so)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol(spk):
    hdr = open(os.path.join(ROOT, "include", "spike_b200.h")).read()
    decls = sorted(set(re.findall(r"\b(spk_[a-z0-9_]+)\s*\(", hdr)))
    assert len(decls) >= 25
    lib = spk.lib()
    missing = [d for d in decls if not hasattr(lib, d)]
    assert not missing, missing


def test_distribute_threads_reference_configurations(spk):
    K = spk.PartitionKind
    p4 = spk.distribute_threads(4)
    assert p4.p == 4 and p4.kinds == [K.FirstLast, K.InnerSingle, K.InnerSingle, K.FirstLast]
    assert p4.idle_threads == 0
    assert spk.distribute_threads(5).kinds == [K.FirstLast, K.InnerDual, K.InnerSingle, K.FirstLast]
    p6 = spk.distribute_threads(6)
    assert p6.kinds == [K.FirstLast, K.InnerDual, K.InnerDual, K.FirstLast] and p6.idle_threads == 0
    p7 = spk.distribute_threads(7)
    assert p7.kinds == p6.kinds and p7.idle_threads == 1 and p7.threads_used == 6
    assert spk.distribute_threads(2).kinds == [K.FirstLast, K.FirstLast]
    p1 = spk.distribute_threads(1)
    assert p1.p == 1 and p1.threads_used == 1
    with pytest.raises(ValueError):
        spk.distribute_threads(0)


def test_distribute_threads_invariants(spk):
    for t in range(2, 65):
        plan = spk.distribute_threads(t)
        p = plan.p
        assert p & (p - 1) == 0 and p <= t < 2 * p
        r, q = plan.dual_count(), plan.single_count()
        assert q + r == p and plan.threads_used == q + 2 * r
        assert plan.idle_threads == (1 if (t & (t + 1)) == 0 and t > 2 else 0)
        assert plan.idle_threads + plan.threads_used == t


def test_compute_ratios_limits(spk):
    r12, r13 = spk.compute_ratios(1.7, 1 << 20, 1)
    assert abs(r12 - 1.0) < 1e-5 and abs(r13 - 2.0) < 1e-5
    r12, r13 = spk.compute_ratios(4.0 / 3.0, 0, 8)
    assert abs(r12 - 1.5) < 1e-12 and abs(r13 - 3.0) < 1e-12
    r12, r13 = spk.compute_ratios(1.0, 8, 8)
    assert abs(r13 - 2.25) < 1e-12 and abs(r12 - 1.125) < 1e-12
    with pytest.raises(ValueError):
        spk.compute_ratios(0.0, 1, 1)


def test_compute_sizes_known_answers(spk):
    assert spk.compute_sizes(1200, spk.distribute_threads(4), 1.0, 2.0, 1, 1) == [400, 200, 200, 400]
    assert spk.compute_sizes(1000, spk.distribute_threads(2), 1.0, 2.0, 1, 1) == [500, 500]
    assert spk.compute_sizes(1000, spk.distribute_threads(6), 1.15, 2.3, 1, 1) == [267, 233, 233, 267]


def test_make_plan_degradation(spk):
    serial = spk.make_plan(64, 16, 16, 8, 1.0, 2.0)
    assert serial.p == 1 and serial.bounds == [0, 64]
    d = spk.make_plan(40, 2, 2, 8, 1.0, 2.0)
    assert d.p == 4 and d.n() == 40 and d.dual_count() == 2
    assert spk.make_plan(64, 4, 4, 8, 1.0, 2.0).p == 2
    full = spk.make_plan(4096, 4, 4, 8, 1.0, 2.0)
    assert full.p == 8 and full.n() == 4096


def test_make_plan_matches_golden(spk):
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    for row in g["plans"]:
        n, k, t, nrhs, p, tu, idle = [int(x) for x in row[:7]]
        r12, r13 = spk.compute_ratios(1.0, nrhs, k)
        pl = spk.make_plan(n, k, k, t, r12, r13)
        assert (pl.p, pl.threads_used, pl.idle_threads) == (p, tu, idle)
        exp = [int(b) for b in row[7:] if b >= 0]
        assert pl.bounds[:len(exp)] == exp


@pytest.mark.parametrize("n,k,p", [(10**6, 160, 0), (10**6, 64, 0), (10**5, 16, 0), (5000, 8, 7),
                                   (1000, 16, 13), (64, 1, 3)])
def test_gpu_plan_properties(spk, n, k, p):
    pl = spk.gpu_plan(n, k, k, 1, False, p)
    assert pl.bounds[0] == 0 and pl.bounds[-1] == n and len(pl.bounds) == pl.p + 1
    sizes = [pl.size(i) for i in range(pl.p)]
    assert all(s >= 2 * k + 1 for s in sizes) or pl.p == 1
    if p:
        assert pl.p == p
    assert max(sizes) - min(sizes) <= 1 + (n % pl.p > 0) * n // pl.p  # equal partitions


def test_banded_matrix_mirror(spk):
    a = spk.BandedMatrix(5, 1, 2)
    a.set(2, 3, 4.0)
    assert a.at(2, 3) == 4.0 and a.at(4, 0) == 0.0
    with pytest.raises(IndexError):
        a.set(4, 0, 1.0)
    with pytest.raises(IndexError):
        a.at(5, 0)
    with pytest.raises(ValueError):
        spk.BandedMatrix(0, 0, 0)
    with pytest.raises(ValueError):
        spk.BandedMatrix(3, 3, 0)
    i3 = spk.BandedMatrix.identity(3)
    assert np.array_equal(i3.dense(), np.eye(3))


def test_no_cpu_fallback_without_library(monkeypatch, tmp_path):
    """The product path fails loudly when the CUDA library is missing."""
    import paper_1811_03559_b200.spike as sp
    monkeypatch.setattr(sp, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(sp, "_lib", None)
    with pytest.raises(ImportError):
        sp.lib()
    # monkeypatch restores LIB_PATH and _lib (no module reload: that would
    # re-create the exception classes other tests match against)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1811_03559_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).lower() or fn == "__init__.py", fn


def test_cpp_api_surface_links(spk, tmp_path):
    """The reference's C++ entry points of the path (factorize / solve /
    transpose_solve, the planner, the 2x2 kernel's wrappers, band ops and I/O)
    exist in include/spike and link against libspike_b200.so; nothing is
    called, so no GPU is needed."""
    import shutil
    import subprocess
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("no g++")
    exe = str(tmp_path / "api_surface")
    libdir = os.path.dirname(spk.LIB_PATH)
    subprocess.run([cxx, "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "api_surface.cpp"), "-L" + libdir, "-lspike_b200",
                    "-Wl,-rpath," + libdir, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "api surface ok" in r.stdout
