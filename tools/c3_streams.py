"""C3 step with the forward and the transpose solve on two streams (the
C-ABI's concurrent-solve contract) vs one stream: CUDA-event timing."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_1811_03559_b200 as spk

n, k, nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, 160, 160
dev = torch.device("cuda", 0)
s1 = torch.cuda.current_stream()
s2 = torch.cuda.Stream()
band = torch.empty((n, 2 * k + 1), dtype=torch.float64, device=dev)
F = torch.empty((nrhs, n), dtype=torch.float64, device=dev)
X = torch.empty_like(F)
XT = torch.empty_like(F)
spk.generate_band_device(20181108, n, k, k, 1.5, band.data_ptr(), s1.cuda_stream)
spk.generate_rhs_device(20181109, n, nrhs, F.data_ptr(), n, s1.cuda_stream)
plan = spk.gpu_plan(n, k, k, nrhs, False, 0)
L = spk.lib()
st, keep = spk.spike._plan_struct(plan)
o = spk.spike._Opts(0, spk.FactorOptions().boost_eps)


def step(two):
    h = C.c_void_p()
    spk.spike._check(L.spk_factorize(C.c_void_p(band.data_ptr()), 1, n, k, k, C.byref(st), C.byref(o),
                                      s1.cuda_stream, C.byref(h)))
    spk.spike._check(L.spk_solve(h, 0, C.c_void_p(F.data_ptr()), n, nrhs, C.c_void_p(X.data_ptr()), n, 1,
                                 s1.cuda_stream, None))
    ss = s2 if two else s1
    spk.spike._check(L.spk_solve(h, 1, C.c_void_p(F.data_ptr()), n, nrhs, C.c_void_p(XT.data_ptr()), n, 1,
                                 ss.cuda_stream, None))
    if two:
        e = torch.cuda.Event()
        e.record(s2)
        s1.wait_event(e)
    L.spk_fact_destroy(h)


for two in (False, True, False, True):
    for _ in range(3):
        step(two)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    for _ in range(5):
        step(two)
    e1.record(s1)
    torch.cuda.synchronize()
    print(f"two streams={two}: {e0.elapsed_time(e1) / 5:.3f} ms/step", flush=True)
