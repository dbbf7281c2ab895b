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
for it in range(6):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    fact = spk.factorize_device(band.data_ptr(), n, k, k, plan, spk.FactorOptions(), s)
    e[1].record()
    spk.solve_device(fact, F.data_ptr(), n, nrhs, X.data_ptr(), n, False, s)
    e[2].record()
    torch.cuda.synchronize()
    print(f"p={plan.p} engine={spk.fact_engine(fact)} factor {e[0].elapsed_time(e[1]):.3f} ms "
          f"solve {e[1].elapsed_time(e[2]):.3f} ms")
