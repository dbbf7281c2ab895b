import sys, numpy as np
if len(sys.argv) > 1: import torch; torch.cuda.init(); torch.zeros(1, device="cuda")
sys.path.insert(0, "/root/repo")
import paper_1811_03559_b200 as spk
from oracle.oracle import Oracle
o = Oracle("/root/repo/oracle/liboracle.so")
n, kl, ku, p, dd, nrhs = 3000, 1, 1, 17, 1.5, 3
band = o.generate_band(3100 + n + kl + 7 * ku, n, kl, ku, dd)
F = np.asfortranarray(o.generate_rhs(3200 + n, n, nrhs))
a = spk.BandedMatrix(n, kl, ku, band)
plan = spk.gpu_plan(n, kl, ku, nrhs, False, p)
print("plan", plan.p, flush=True)
fact = spk.factorize(a, plan)
print("factorized", flush=True)
x1 = spk.solve(fact, F)
print("solved", flush=True)
print("engine", spk.fact_engine(fact), "nan1", np.isnan(x1).sum())
f2 = spk.factorize(a, plan)
x2 = spk.solve(f2, F)
print("nan2", np.isnan(x2).sum(), "eq", np.array_equal(x1, x2))
x3 = spk.solve(fact, F)
print("nan3", np.isnan(x3).sum(), "eq", np.array_equal(x1, x3), np.where(np.isnan(x3))[0][:10])
