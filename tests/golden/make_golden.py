"""Generate the golden fixtures that pin the CPU oracle (oracle/spike_oracle.c).

Runs the UNMODIFIED reference library (oracle/_ref/libspike_ref.so, compiled
from /root/reference/proj/src by oracle/Makefile) on seeded inputs from the
shared generator (include/spike_b200_gen.h) and stores inputs' seeds, plans,
tips, solutions, sweep counts and reduced-system solutions in
tests/golden/golden.npz.  Only needs to run where /root/reference exists; the
fixtures are committed so the GPU box and the CPU test suite never read the
reference tree.

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, Reference, build  # noqa: E402

# (name, n, kl, ku, dd, nrhs, t, pivoting) ; dd <= 0: no dominance (U[-1,1] diagonal)
CASES = [
    ("c1_small", 4000, 16, 16, 2.0, 1, 4, False),
    ("c2_small", 3000, 8, 8, 1.1, 1, 3, False),
    ("c3_small", 2048, 12, 12, 1.5, 12, 8, False),
    ("c4_small", 3000, 6, 6, -1.0, 4, 4, True),
    ("asym", 600, 2, 5, 1.5, 3, 6, False),
    ("asym_piv", 600, 5, 2, 1.5, 3, 6, True),
    ("dual_mix", 4096, 8, 8, 1.5, 4, 12, False),
    ("serial", 300, 3, 3, 1.5, 2, 1, False),
    ("k1", 512, 1, 1, 1.5, 3, 5, True),
]
SEED = 20181108


def main():
    build(with_ref=True)
    ref = Reference.load()
    o = Oracle()
    out = {}
    for (name, n, kl, ku, dd, nrhs, t, piv) in CASES:
        k = max(kl, ku)
        band = o.generate_band(SEED, n, kl, ku, dd)
        F = o.generate_rhs(SEED + 1, n, nrhs)
        r12, r13 = ref.compute_ratios(1.0, nrhs, k)
        plan = ref.make_plan(n, kl, ku, t, r12, r13)
        fact = ref.factorize_t(band, n, kl, ku, t, r12, r13, piv)
        x, sw, cc = fact.solve(F, False)
        xt, swt, cct = fact.solve(F, True)
        pre = name + "/"
        out[pre + "shape"] = np.array([n, kl, ku, nrhs, t, int(piv)], dtype=np.int64)
        out[pre + "dd"] = np.array([dd])
        out[pre + "bounds"] = np.array(plan["bounds"], dtype=np.int64)
        out[pre + "kinds"] = np.array(plan["kinds"], dtype=np.int64)
        out[pre + "band_checksum"] = np.array([band.sum(), np.abs(band).sum()])
        out[pre + "x"] = x
        out[pre + "xt"] = xt
        out[pre + "sweeps"] = np.array(sw, dtype=np.int64)
        out[pre + "sweeps_t"] = np.array(swt, dtype=np.int64)
        out[pre + "couplings"] = np.array([cc, cct], dtype=np.int64)
        out[pre + "factor_sweeps"] = np.array(fact.factor_sweeps(), dtype=np.int64)
        out[pre + "levels"] = np.array([fact.levels, fact.boost_count], dtype=np.int64)
        for w in ("vt", "vb", "wt", "wb", "bhat", "chat"):
            out[pre + w] = np.stack([fact.tip(w, i) for i in range(fact.p)])
        out[pre + "x_oracle_solve"] = ref.oracle_solve(band, n, kl, ku, F, False, True)
        out[pre + "relres"] = np.array([ref.relative_residual(band, n, kl, ku, x, F, False),
                                        ref.relative_residual(band, n, kl, ku, xt, F, True)])
        print(name, "p", fact.p, "levels", fact.levels, "relres", out[pre + "relres"])
    # diagonal boosting (kernels.cpp:104-109): exact zeros on the first pivot
    # of every partition (the UL partition's first pivot is its last row), so
    # the boost count is known (one per partition) and the boosted
    # factorization is pinned: its solution and the reference's
    # iterative_refine (solve.cpp:404-432) from x0 = 0 on it
    n, k, nrhs, t = 4000, 8, 2, 4
    band = o.generate_band(SEED + 77, n, k, k, 1.5)
    F = o.generate_rhs(SEED + 78, n, nrhs)
    r12, r13 = ref.compute_ratios(1.0, nrhs, k)
    plan = ref.make_plan(n, k, k, t, r12, r13)
    b = plan["bounds"]
    for r in [0] + b[1:-2] + [n - 1]:
        band[r, k] = 0.0  # A(r, r): packed row ku of column r
    fact = ref.factorize_t(band, n, k, k, t, r12, r13, False)
    x, _, _ = fact.solve(F, False)
    xt, _, _ = fact.solve(F, True)
    xr, its, conv, stag, res = fact.iterative_refine(F, np.zeros((n, nrhs)), 10, 1e-14, False)
    xrt, itst, convt, stagt, rest = fact.iterative_refine(F, np.zeros((n, nrhs)), 10, 1e-14, True)
    pre = "boost/"
    out[pre + "shape"] = np.array([n, k, k, nrhs, t, 0], dtype=np.int64)
    out[pre + "band"] = band
    out[pre + "F"] = F
    out[pre + "bounds"] = np.array(b, dtype=np.int64)
    out[pre + "boost_count"] = np.array([fact.boost_count], dtype=np.int64)
    out[pre + "x"] = x
    out[pre + "xt"] = xt
    out[pre + "x_refined"] = xr
    out[pre + "xt_refined"] = xrt
    out[pre + "refine"] = np.array([[its, conv, stag, res], [itst, convt, stagt, rest]])
    print("boost", "p", fact.p, "boosts", fact.boost_count, "refine", out[pre + "refine"])
    # reduced-system brute force vectors (test_acceptance.cpp:109-151 shape)
    rng = np.random.default_rng(4242)
    for p in (2, 4, 8):
        for k in (1, 2, 3):
            tips = [rng.random((p, k, k)) - 0.5 for _ in range(4)]
            y = rng.random((2 * p * k, 2))
            z, c = ref.reduced_solve_tips(*tips, p, k, y, False)
            zt, ct = ref.reduced_solve_tips(*tips, p, k, y, True)
            pre = f"reduced_p{p}_k{k}/"
            for nm, arr in zip(("vt", "vb", "wt", "wb"), tips):
                out[pre + nm] = arr
            out[pre + "y"] = y
            out[pre + "z"] = z
            out[pre + "zt"] = zt
            out[pre + "couplings"] = np.array([c, ct], dtype=np.int64)
    # planner known answers (partition.cpp) for a spread of inputs
    plans = []
    for (n, k, t, nrhs) in [(1000, 4, 5, 1), (800, 4, 4, 4), (100000, 16, 4, 1), (1000000, 64, 3, 1),
                            (1000000, 160, 8, 160), (100, 3, 1, 2), (64, 2, 14, 1), (4096, 8, 12, 4),
                            (1000000, 64, 64, 4), (200, 40, 16, 1)]:
        r12, r13 = ref.compute_ratios(1.0, nrhs, k)
        pl = ref.make_plan(n, k, k, t, r12, r13)
        plans.append([n, k, t, nrhs, pl["p"], pl["threads_used"], pl["idle_threads"]] + pl["bounds"][:17]
                     + [-1] * (17 - len(pl["bounds"][:17])))
    out["plans"] = np.array(plans, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"))
    write_spkb_fixtures(ref, o)


# .spkb files written by the reference's own band_io.cpp (write_matrix,
# MatrixFormat::Spkb): the byte-level contract of spk_spkb_load / _store
SPKB_CASES = [("ref_n300_kl3_ku5.spkb", 300, 3, 5, 1.5), ("ref_n1_kl0_ku0.spkb", 1, 0, 0, 2.0),
              ("ref_n257_kl16_ku2.spkb", 257, 16, 2, 1.2)]


def write_spkb_fixtures(ref, o):
    for (fname, n, kl, ku, dd) in SPKB_CASES:
        band = o.generate_band(SEED + n, n, kl, ku, dd)
        path = os.path.join(HERE, fname)
        ref.write_spkb(band, n, kl, ku, path)
        rn, rkl, rku, back = ref.read_spkb(path)
        assert (rn, rkl, rku) == (n, kl, ku) and np.array_equal(back, band)
        print("wrote", path)


if __name__ == "__main__":
    main()
