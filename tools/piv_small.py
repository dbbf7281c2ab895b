"""Small pivoted factorizations (symmetric and asymmetric bands) against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_03559_b200 as spk  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

o = Oracle()
cases = [(200, 3, 3, 2), (2000, 8, 8, 4), (1500, 5, 8, 2), (1500, 8, 5, 2), (1500, 2, 7, 3), (3000, 16, 16, 5)]
for (n, kl, ku, p) in cases:
    band = o.generate_band(5, n, kl, ku, 1.2)  # dominant: SPIKE's partition coupling is stable
    F = np.asfortranarray(o.generate_rhs(6, n, 2))
    a = spk.BandedMatrix(n, kl, ku, band)
    fact = spk.factorize(a, spk.gpu_plan(n, kl, ku, 2, True, p), spk.FactorOptions(pivoting=True))
    X = spk.solve(fact, F)
    print(n, kl, ku, p, "res", o.relative_residual(band, n, kl, ku, X, F, False), flush=True)
