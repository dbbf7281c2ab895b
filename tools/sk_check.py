"""Small-k engine vs the general engine on one plan: packed factor, 1/u,
level-0 tips, level spikes, solution (debug aid)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1811_03559_b200 as spk
from oracle.oracle import Oracle

o = Oracle("oracle/liboracle.so")
n, kl, ku, p, dd = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])) \
    if len(sys.argv) > 5 else (20000, 16, 16, 104, 2.0)
band = o.generate_band(3100 + n + kl + 7 * ku, n, kl, ku, dd)
F = np.asfortranarray(o.generate_rhs(3200 + n, n, 1))
a = spk.BandedMatrix(n, kl, ku, band)
plan = spk.gpu_plan(n, kl, ku, 1, False, p)
f = spk.factorize(a, plan)
with spk.generic_path():
    g = spk.factorize(a, plan)
print("engines", spk.fact_engine(f), spk.fact_engine(g), "p", plan.p)
L = spk.lib()
L.spk_fact_dump.restype = C.c_int64
L.spk_fact_dump.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]


def dump(fc, w):
    sz = L.spk_fact_dump(fc._h, w, None)
    out = np.zeros(sz)
    L.spk_fact_dump(fc._h, w, out.ctypes.data)
    return out


for w, name in ((0, "fac"), (2, "dinv"), (1, "tfac")):
    x, y = dump(f, w), dump(g, w)
    d = np.abs(x - y)
    print(name, "maxdiff", d.max(), "at", int(d.argmax()), "of", len(d))
for w in ("vt", "vb", "wt", "wb", "bhat", "chat"):
    worst = max((np.abs(getattr(f, w)[i] - getattr(g, w)[i]).max(), i) for i in range(plan.p))
    print(w, "max diff, part", worst)
for l in range(f.levels.levels()):
    for u in range(len(f.levels.v[l])):
        dv = np.abs(np.asarray(f.levels.v[l][u]) - np.asarray(g.levels.v[l][u])).max()
        dw = np.abs(np.asarray(f.levels.w[l][u]) - np.asarray(g.levels.w[l][u])).max()
        if dv > 1e-12 or dw > 1e-12:
            print("level", l, "unit", u, "dv", dv, "dw", dw)
X = spk.solve(f, F)
Xg = spk.solve(g, F)
print("solve diff", np.abs(X - Xg).max())
