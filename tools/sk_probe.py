"""Time the small-k engine's kernels on BASELINE C1 (n=1e5, k=16, nrhs=1):
CUDA events around factorize_device / solve_device, optional partition count."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1811_03559_b200 as spk

n, k, nrhs = 100_000, 16, 1
p = int(sys.argv[1]) if len(sys.argv) > 1 else 0
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream().cuda_stream
band = torch.empty((n, 2 * k + 1), dtype=torch.float64, device=dev)
F = torch.empty((nrhs, n), dtype=torch.float64, device=dev)
X = torch.empty_like(F)
spk.generate_band_device(20181108, n, k, k, 2.0, band.data_ptr(), s)
spk.generate_rhs_device(20181109, n, nrhs, F.data_ptr(), n, s)
plan = spk.gpu_plan(n, k, k, nrhs, False, p)
import time
for it in range(6):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    h0 = time.perf_counter()
    fact = spk.factorize_device(band.data_ptr(), n, k, k, plan, spk.FactorOptions(), s)
    h1 = time.perf_counter()
    e[1].record()
    spk.solve_device(fact, F.data_ptr(), n, nrhs, X.data_ptr(), n, False, s)
    h2 = time.perf_counter()
    e[2].record()
    torch.cuda.synchronize()
    print(f"p={plan.p} engine={spk.fact_engine(fact)} factor {e[0].elapsed_time(e[1]):.3f} ms "
          f"solve {e[1].elapsed_time(e[2]):.3f} ms  host: factorize {1e3 * (h1 - h0):.3f} ms solve {1e3 * (h2 - h1):.3f} ms",
          flush=True)

# the raw C-ABI loop (what bench.py times): factorize + solve + destroy per
# step, no host waits; CUDA events around 20 steps
import ctypes as C
L = spk.lib()
st, keep = spk.spike._plan_struct(plan)
o = spk.spike._Opts(0, spk.FactorOptions().boost_eps)


def step():
    h = C.c_void_p()
    spk.spike._check(L.spk_factorize(C.c_void_p(band.data_ptr()), 1, n, k, k, C.byref(st), C.byref(o), s,
                                      C.byref(h)))
    spk.spike._check(L.spk_solve(h, 0, C.c_void_p(F.data_ptr()), n, nrhs, C.c_void_p(X.data_ptr()), n, 1, s, None))
    L.spk_fact_destroy(h)


for _ in range(5):
    step()
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    for _ in range(20):
        step()
    e1.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"C-ABI loop: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/step (host enqueue {1e6 * (h1 - h0) / 20:.1f} us/step)")
