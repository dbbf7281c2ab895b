"""Phase timeline of the small-k engine's cooperative kernels (globaltimer
stamps through spk_debug_set_trace): per level phase, the slowest CTA's task
A, task B and barrier wait, in microseconds."""
import sys

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
tr = torch.zeros(2 * 65536, dtype=torch.int64, device=dev)
L = spk.lib()
import ctypes as C
L.spk_debug_set_trace.argtypes = [C.c_void_p]
for it in range(3):
    L.spk_debug_set_trace(tr.data_ptr() if it == 2 else None)
    tr.zero_()
    fact = spk.factorize_device(band.data_ptr(), n, k, k, plan, spk.FactorOptions(), s)
    spk.solve_device(fact, F.data_ptr(), n, nrhs, X.data_ptr(), n, False, s)
    torch.cuda.synchronize()
L.spk_debug_set_trace(None)
t = tr.cpu().numpy()
sms = 148
for name, base in (("factor levels", 0), ("solve", 65536)):
    seg = t[base:base + 60000]
    a = seg[:len(seg) // (sms * 4) * sms * 4].reshape(-1, sms, 4)
    nph = int((a[:, :, 0] > 0).any(axis=1).sum())
    if nph == 0:
        continue
    t0 = a[0, :, 0][a[0, :, 0] > 0].min()
    print(f"{name}: plan p={plan.p}, {nph} phases")
    for ph in range(nph):
        r = a[ph]
        ok = r[:, 0] > 0
        if not ok.any():
            continue
        st = (r[ok, 0].min() - t0) / 1e3
        ta = (r[ok, 1] - r[ok, 0]).max() / 1e3 if (r[ok, 1] > 0).all() else float("nan")
        tb = (r[ok, 2] - r[ok, 1]).max() / 1e3 if (r[ok, 2] > 0).all() else float("nan")
        end = (r[ok, 3].max() - t0) / 1e3 if (r[ok, 3] > 0).any() else float("nan")
        print(f"  phase {ph:2d}: start {st:7.2f} us  taskA max {ta:6.2f}  taskB max {tb:6.2f}  barrier out {end:7.2f}")

