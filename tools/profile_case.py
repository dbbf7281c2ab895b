"""One factorize + solve (+ transpose) on a chosen shape, for ncu / quick timing.

  python tools/profile_case.py --n 200000 --k 160 --nrhs 160 [--piv] [--transpose] [--p P] [--reps R]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1811_03559_b200 as spk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200000)
    ap.add_argument("--k", type=int, default=160)
    ap.add_argument("--nrhs", type=int, default=160)
    ap.add_argument("--dd", type=float, default=1.5)
    ap.add_argument("--piv", action="store_true")
    ap.add_argument("--transpose", action="store_true")
    ap.add_argument("--p", type=int, default=0)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--prof", action="store_true", help="print per-class device times")
    ap.add_argument("--factor-only", action="store_true", help="no solves")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n, k, r = a.n, a.k, a.nrhs
    band = torch.empty((n, 2 * k + 1), dtype=torch.float64, device=dev)
    F = torch.empty((r, n), dtype=torch.float64, device=dev)
    X = torch.empty_like(F)
    s = torch.cuda.current_stream().cuda_stream
    spk.generate_band_device(20181108, n, k, k, a.dd, band.data_ptr(), s)
    spk.generate_rhs_device(20181109, n, r, F.data_ptr(), n, s)
    plan = spk.gpu_plan(n, k, k, r, a.piv, a.p)
    opts = spk.FactorOptions(pivoting=a.piv)
    if a.prof:
        spk.lib().spk_profile_enable(1)
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fact = spk.factorize_device(band.data_ptr(), n, k, k, plan, opts, s)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if not a.factor_only:
            spk.solve_device(fact, F.data_ptr(), n, r, X.data_ptr(), n, False, s)
        if a.transpose and not a.factor_only:
            spk.solve_device(fact, F.data_ptr(), n, r, X.data_ptr(), n, True, s)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"p={plan.p} factor {1e3 * (t1 - t0):.2f} ms  solve(s) {1e3 * (t2 - t1):.2f} ms")
        del fact
    if a.prof:
        import ctypes as C
        L = spk.lib()
        L.spk_profile_read.restype = C.c_char_p
        L.spk_profile_read.argtypes = [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        for c in range(L.spk_profile_classes()):
            ms, fl, by, ln = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
            name = L.spk_profile_read(c, C.byref(ms), C.byref(fl), C.byref(by), C.byref(ln)).decode()
            if ln.value:
                print(f"  {name:12s} {ms.value / a.reps:9.3f} ms  {ln.value // a.reps:4d} launches  "
                      f"{fl.value / max(ms.value, 1e-9) / 1e9:8.1f} TF/s  {by.value / max(ms.value, 1e-9) / 1e6:8.1f} GB/s")


if __name__ == "__main__":
    main()
