"""PCIe / host-path timing probe for the e2e leg (C3 shapes)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1811_03559_b200 as spk  # noqa: E402

n, k, r = 1_000_000, 160, 160
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream()
hF = torch.empty((r, n), dtype=torch.float64).pin_memory()
hX = torch.empty_like(hF).pin_memory()
dF = torch.empty((r, n), dtype=torch.float64, device=dev)
dX = torch.empty_like(dF)
hF.uniform_(-1, 1)


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps


up = torch.cuda.Stream()
down = torch.cuda.Stream()
print("H2D 1.28 GB   %.1f ms" % t(lambda: dF.copy_(hF, non_blocking=True)))
print("D2H 1.28 GB   %.1f ms" % t(lambda: hX.copy_(dX, non_blocking=True)))


def both():
    with torch.cuda.stream(up):
        dF.copy_(hF, non_blocking=True)
    with torch.cuda.stream(down):
        hX.copy_(dX, non_blocking=True)
    up.synchronize()
    down.synchronize()


print("H2D+D2H conc. %.1f ms" % t(both))
band = torch.empty((n, 2 * k + 1), dtype=torch.float64, device=dev)
spk.generate_band_device(1, n, k, k, 1.5, band.data_ptr(), s.cuda_stream)
plan = spk.gpu_plan(n, k, k, r)
fact = spk.factorize_device(band.data_ptr(), n, k, k, plan, spk.FactorOptions(), s.cuda_stream)
L = spk.lib()
print("solve device  %.1f ms" % t(lambda: spk.solve_device(fact, dF.data_ptr(), n, r, dX.data_ptr(), n, False,
                                                           s.cuda_stream)))
print("solve host    %.1f ms" % t(lambda: spk.spike._check(L.spk_solve(fact._h, 0, hF.data_ptr(), n, r, hX.data_ptr(),
                                                                        n, 0, s.cuda_stream, None))))
print("tsolve host   %.1f ms" % t(lambda: spk.spike._check(L.spk_solve(fact._h, 1, hF.data_ptr(), n, r, hX.data_ptr(),
                                                                        n, 0, s.cuda_stream, None))))
hband = band.cpu().pin_memory()
print("factor host   %.1f ms" % t(lambda: spk.factorize(spk.BandedMatrix(n, k, k, hband.numpy()), plan), reps=2))
