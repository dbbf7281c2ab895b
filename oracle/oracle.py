"""ctypes access to the CPU checkers — TEST INFRASTRUCTURE ONLY.

* ``Oracle``    : oracle/liboracle.so, the C restatement (spike_oracle.c) of the
                  reference recursive-SPIKE path.
* ``Reference`` : oracle/_ref/libspike_ref.so, the unmodified reference library
                  (/root/reference/proj/src) behind ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
timed CPU baseline.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def build(with_ref: bool | None = None) -> None:
    """Compile liboracle.so (and oracle/_ref when the reference tree exists)."""
    targets = ["oracle"]
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj/src")
    if with_ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


class _Plan(C.Structure):
    _fields_ = [("p", C.c_int), ("bounds", _ip), ("kinds", _ip), ("threads_used", C.c_int),
                ("idle_threads", C.c_int), ("r12", C.c_double), ("r13", C.c_double)]


def band_ld(kl, ku):
    return kl + ku + 1


class Oracle:
    """The C restatement; band arrays are (ld, n) column-major = numpy (n, ld) C-order."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(with_ref=False)
        L = C.CDLL(path)
        self.L = L
        L.orc_make_plan.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.POINTER(_Plan)]
        L.orc_plan_from_bounds.argtypes = [C.c_int, _ip, C.POINTER(_Plan)]
        L.orc_plan_free.argtypes = [C.POINTER(_Plan)]
        L.orc_compute_ratios.argtypes = [C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.orc_factorize.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.POINTER(_Plan), C.c_int,
                                    C.c_double]
        L.orc_factorize.restype = C.c_void_p
        L.orc_fact_free.argtypes = [C.c_void_p]
        for fn in ("orc_fact_p", "orc_fact_k", "orc_fact_boost_count", "orc_fact_levels"):
            getattr(L, fn).argtypes = [C.c_void_p]
        L.orc_fact_factor_sweeps.argtypes = [C.c_void_p, _lp]
        L.orc_fact_tip.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.orc_solve.argtypes = [C.c_void_p, _dp, C.c_int, C.c_int, _dp, _lp, _lp]
        L.orc_reduced_solve_tips.argtypes = [_dp, _dp, _dp, _dp, C.c_int, C.c_int, _dp, C.c_int,
                                             C.c_int, _lp]
        L.orc_oracle_solve.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                                       C.c_int, _dp]
        L.orc_condition_estimate_1norm.argtypes = [_dp, C.c_int, C.c_int, C.c_int]
        L.orc_condition_estimate_1norm.restype = C.c_double
        L.orc_band_matmul.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int, C.c_int, _dp]
        L.orc_relative_residual.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int,
                                            C.c_int]
        L.orc_relative_residual.restype = C.c_double
        L.orc_backward_error_inf.argtypes = L.orc_relative_residual.argtypes
        L.orc_backward_error_inf.restype = C.c_double
        L.orc_generate_band.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_double, _dp]
        L.orc_generate_rhs.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
        L.orc_last_error.restype = C.c_char_p

    # ---- inputs
    def generate_band(self, seed, n, kl, ku, dd):
        a = np.zeros((n, kl + ku + 1))
        self.L.orc_generate_band(seed, n, kl, ku, dd, _d(a))
        return a

    def generate_rhs(self, seed, n, ncols):
        f = np.zeros((ncols, n))
        self.L.orc_generate_rhs(seed, n, ncols, _d(f))
        return f.T  # (n, ncols) Fortran-ordered view

    # ---- planning
    def compute_ratios(self, K, nrhs, k):
        a, b = C.c_double(), C.c_double()
        self.L.orc_compute_ratios(K, nrhs, k, C.byref(a), C.byref(b))
        return a.value, b.value

    def make_plan(self, n, kl, ku, t, r12, r13):
        pl = _Plan()
        if self.L.orc_make_plan(n, kl, ku, t, r12, r13, C.byref(pl)) != 0:
            raise ValueError(self.L.orc_last_error().decode())
        out = dict(p=pl.p, bounds=[pl.bounds[i] for i in range(pl.p + 1)],
                   kinds=[pl.kinds[i] for i in range(pl.p)], threads_used=pl.threads_used,
                   idle_threads=pl.idle_threads)
        self.L.orc_plan_free(C.byref(pl))
        return out

    # ---- factor / solve
    def factorize(self, band, n, kl, ku, bounds, pivoting=False,
                  boost_eps=float(np.sqrt(np.finfo(float).eps))):
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        pl = _Plan()
        self.L.orc_plan_from_bounds(len(b) - 1, b.ctypes.data_as(_ip), C.byref(pl))
        band = np.ascontiguousarray(band, dtype=np.float64)
        h = self.L.orc_factorize(_d(band), n, kl, ku, C.byref(pl), int(pivoting), boost_eps)
        self.L.orc_plan_free(C.byref(pl))
        if not h:
            raise RuntimeError(self.L.orc_last_error().decode())
        return OracleFact(self, h, n, len(b) - 1, max(kl, ku))

    def oracle_solve(self, band, n, kl, ku, F, transpose=False, pivoting=True):
        F = np.asfortranarray(F, dtype=np.float64)
        X = np.zeros_like(F, order="F")
        band = np.ascontiguousarray(band, dtype=np.float64)
        rc = self.L.orc_oracle_solve(_d(band), n, kl, ku, _d(F), F.shape[1], int(transpose),
                                     int(pivoting), _d(X))
        if rc:
            raise RuntimeError(self.L.orc_last_error().decode())
        return X

    def reduced_solve_tips(self, vt, vb, wt, wb, p, k, z, transpose=False):
        z = np.asfortranarray(z, dtype=np.float64).copy(order="F")
        cnt = C.c_long(0)
        arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (vt, vb, wt, wb)]
        self.L.orc_reduced_solve_tips(*[_d(a) for a in arrs], p, k, _d(z), z.shape[1],
                                      int(transpose), C.byref(cnt))
        return z, cnt.value

    def cond1(self, band, n, kl, ku):
        band = np.ascontiguousarray(band, dtype=np.float64)
        return self.L.orc_condition_estimate_1norm(_d(band), n, kl, ku)

    def matmul(self, band, n, kl, ku, X, transpose=False):
        X = np.asfortranarray(X, dtype=np.float64)
        Y = np.zeros_like(X, order="F")
        band = np.ascontiguousarray(band, dtype=np.float64)
        self.L.orc_band_matmul(_d(band), n, kl, ku, _d(X), X.shape[1], int(transpose), _d(Y))
        return Y

    def relative_residual(self, band, n, kl, ku, X, F, transpose=False):
        X = np.asfortranarray(X, dtype=np.float64)
        F = np.asfortranarray(F, dtype=np.float64)
        band = np.ascontiguousarray(band, dtype=np.float64)
        return self.L.orc_relative_residual(_d(band), n, kl, ku, _d(X), _d(F), X.shape[1],
                                            int(transpose))

    def backward_error(self, band, n, kl, ku, X, F, transpose=False):
        X = np.asfortranarray(X, dtype=np.float64)
        F = np.asfortranarray(F, dtype=np.float64)
        band = np.ascontiguousarray(band, dtype=np.float64)
        return self.L.orc_backward_error_inf(_d(band), n, kl, ku, _d(X), _d(F), X.shape[1],
                                             int(transpose))


class OracleFact:
    TIPS = ("vt", "vb", "wt", "wb", "bhat", "chat")

    def __init__(self, o, h, n, p, k):
        self.o, self.h, self.n, self.p, self.k = o, h, n, p, k

    def __del__(self):
        try:
            self.o.L.orc_fact_free(self.h)
        except Exception:
            pass

    @property
    def levels(self):
        return self.o.L.orc_fact_levels(self.h)

    @property
    def boost_count(self):
        return self.o.L.orc_fact_boost_count(self.h)

    def factor_sweeps(self):
        out = (C.c_long * self.p)()
        self.o.L.orc_fact_factor_sweeps(self.h, out)
        return list(out)

    def tip(self, which, i):
        out = np.zeros((self.k, self.k))
        self.o.L.orc_fact_tip(self.h, self.TIPS.index(which), i, _d(out))
        return out.T  # column-major k x k

    def solve(self, F, transpose=False):
        F = np.asfortranarray(F, dtype=np.float64)
        X = np.zeros_like(F, order="F")
        sw = (C.c_long * self.p)()
        cc = C.c_long(0)
        self.o.L.orc_solve(self.h, _d(F), F.shape[1], int(transpose), _d(X), sw, C.byref(cc))
        return X, list(sw), cc.value


class Reference:
    """The compiled reference library (oracle/_ref); None-safe constructor via ``load``."""

    @staticmethod
    def load():
        path = os.path.join(HERE, "_ref", "libspike_ref.so")
        if not os.path.exists(path):
            return None
        return Reference(path)

    def __init__(self, path):
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_compute_ratios.argtypes = [C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.ref_make_plan.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_int, _ip, _ip, _ip, _ip, _ip]
        L.ref_factorize.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                    C.c_double, C.c_int]
        L.ref_factorize.restype = C.c_void_p
        L.ref_factorize_bounds.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _ip, C.c_int]
        L.ref_factorize_bounds.restype = C.c_void_p
        L.ref_free.argtypes = [C.c_void_p]
        for fn in ("ref_fact_p", "ref_fact_boost_count", "ref_fact_levels"):
            getattr(L, fn).argtypes = [C.c_void_p]
        L.ref_fact_factor_sweeps.argtypes = [C.c_void_p, _lp]
        L.ref_fact_bounds.argtypes = [C.c_void_p, _ip]
        L.ref_fact_tip.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.ref_solve.argtypes = [C.c_void_p, _dp, C.c_int, C.c_int, _dp, _lp, _lp]
        L.ref_reduced_solve_tips.argtypes = [_dp, _dp, _dp, _dp, C.c_int, C.c_int, _dp, C.c_int,
                                             C.c_int, _lp]
        L.ref_oracle_solve.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                                       C.c_int, _dp]
        L.ref_condition_estimate_1norm.argtypes = [_dp, C.c_int, C.c_int, C.c_int]
        L.ref_condition_estimate_1norm.restype = C.c_double
        L.ref_relative_residual.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int,
                                            C.c_int]
        L.ref_relative_residual.restype = C.c_double
        L.ref_time_path.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                                    C.c_double, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _ip]
        L.ref_hw_threads.restype = C.c_int
        L.ref_iterative_refine.argtypes = [C.c_void_p, _dp, C.c_int, _dp, C.c_int, C.c_double, C.c_int, _ip,
                                           _dp]
        L.ref_write_spkb.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_char_p]
        L.ref_read_spkb.argtypes = [C.c_char_p, _ip, _ip, _ip, _dp]

    def err(self):
        return self.L.ref_last_error().decode()

    def write_spkb(self, band, n, kl, ku, path):
        """band_io.cpp write_matrix(..., MatrixFormat::Spkb)"""
        band = np.ascontiguousarray(band, dtype=np.float64)
        if self.L.ref_write_spkb(_d(band), n, kl, ku, path.encode()):
            raise RuntimeError(self.err())

    def read_spkb(self, path):
        """band_io.cpp read_matrix on a .spkb file -> (n, kl, ku, band)"""
        n, kl, ku = C.c_int(), C.c_int(), C.c_int()
        if self.L.ref_read_spkb(path.encode(), C.byref(n), C.byref(kl), C.byref(ku), None):
            raise RuntimeError(self.err())
        band = np.zeros((n.value, kl.value + ku.value + 1))
        self.L.ref_read_spkb(path.encode(), C.byref(n), C.byref(kl), C.byref(ku), _d(band))
        return n.value, kl.value, ku.value, band

    def make_plan(self, n, kl, ku, t, r12, r13):
        cap = 4096
        p = C.c_int()
        tu = C.c_int()
        idle = C.c_int()
        b = (C.c_int * (cap + 1))()
        k = (C.c_int * cap)()
        rc = self.L.ref_make_plan(n, kl, ku, t, r12, r13, cap, C.byref(p), b, k, C.byref(tu),
                                  C.byref(idle))
        if rc:
            raise ValueError(self.err())
        return dict(p=p.value, bounds=list(b[:p.value + 1]), kinds=list(k[:p.value]),
                    threads_used=tu.value, idle_threads=idle.value)

    def compute_ratios(self, K, nrhs, k):
        a, b = C.c_double(), C.c_double()
        self.L.ref_compute_ratios(K, nrhs, k, C.byref(a), C.byref(b))
        return a.value, b.value

    def factorize_bounds(self, band, n, kl, ku, bounds, pivoting=False):
        band = np.ascontiguousarray(band, dtype=np.float64)
        b = np.ascontiguousarray(bounds, dtype=np.int32)
        h = self.L.ref_factorize_bounds(_d(band), n, kl, ku, len(b) - 1, b.ctypes.data_as(_ip),
                                        int(pivoting))
        if not h:
            raise RuntimeError(self.err())
        return RefFact(self, h, n, len(b) - 1, max(kl, ku))

    def factorize_t(self, band, n, kl, ku, t, r12, r13, pivoting=False):
        band = np.ascontiguousarray(band, dtype=np.float64)
        h = self.L.ref_factorize(_d(band), n, kl, ku, t, r12, r13, int(pivoting))
        if not h:
            raise RuntimeError(self.err())
        p = self.L.ref_fact_p(h)
        return RefFact(self, h, n, p, max(kl, ku))

    def oracle_solve(self, band, n, kl, ku, F, transpose=False, pivoting=True):
        F = np.asfortranarray(F, dtype=np.float64)
        X = np.zeros_like(F, order="F")
        band = np.ascontiguousarray(band, dtype=np.float64)
        if self.L.ref_oracle_solve(_d(band), n, kl, ku, _d(F), F.shape[1], int(transpose),
                                   int(pivoting), _d(X)):
            raise RuntimeError(self.err())
        return X

    def reduced_solve_tips(self, vt, vb, wt, wb, p, k, z, transpose=False):
        z = np.asfortranarray(z, dtype=np.float64).copy(order="F")
        cnt = C.c_long(0)
        arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (vt, vb, wt, wb)]
        if self.L.ref_reduced_solve_tips(*[_d(a) for a in arrs], p, k, _d(z), z.shape[1],
                                         int(transpose), C.byref(cnt)):
            raise RuntimeError(self.err())
        return z, cnt.value

    def cond1(self, band, n, kl, ku):
        band = np.ascontiguousarray(band, dtype=np.float64)
        return self.L.ref_condition_estimate_1norm(_d(band), n, kl, ku)

    def relative_residual(self, band, n, kl, ku, X, F, transpose=False):
        X = np.asfortranarray(X, dtype=np.float64)
        F = np.asfortranarray(F, dtype=np.float64)
        band = np.ascontiguousarray(band, dtype=np.float64)
        return self.L.ref_relative_residual(_d(band), n, kl, ku, _d(X), _d(F), X.shape[1],
                                            int(transpose))

    def time_path(self, band, n, kl, ku, F, t, K=1.0, pivoting=False, transpose=False,
                  want_x=False):
        band = np.ascontiguousarray(band, dtype=np.float64)
        F = np.asfortranarray(F, dtype=np.float64)
        tf, ts, tt = C.c_double(), C.c_double(), C.c_double()
        p = C.c_int()
        X = np.zeros_like(F, order="F") if want_x else None
        XT = np.zeros_like(F, order="F") if (want_x and transpose) else None
        rc = self.L.ref_time_path(_d(band), n, kl, ku, _d(F), F.shape[1], t, K, int(pivoting),
                                  int(transpose), C.byref(tf), C.byref(ts), C.byref(tt), _d(X),
                                  _d(XT), C.byref(p))
        if rc:
            raise RuntimeError(self.err())
        return dict(factor=tf.value, solve=ts.value, tsolve=tt.value, p=p.value, X=X, XT=XT)


class RefFact(OracleFact):
    def __del__(self):
        try:
            self.o.L.ref_free(self.h)
        except Exception:
            pass

    @property
    def levels(self):
        return self.o.L.ref_fact_levels(self.h)

    @property
    def boost_count(self):
        return self.o.L.ref_fact_boost_count(self.h)

    def factor_sweeps(self):
        out = (C.c_long * self.p)()
        self.o.L.ref_fact_factor_sweeps(self.h, out)
        return list(out)

    def bounds(self):
        out = (C.c_int * (self.p + 1))()
        self.o.L.ref_fact_bounds(self.h, out)
        return list(out)

    def tip(self, which, i):
        out = np.zeros((self.k, self.k))
        self.o.L.ref_fact_tip(self.h, self.TIPS.index(which), i, _d(out))
        return out.T

    def iterative_refine(self, F, x0, max_iters, tol, transpose=False):
        """solve.cpp:404-432 -> (x, iterations, converged, stagnated, residual)"""
        F = np.asfortranarray(F, dtype=np.float64)
        X = np.asfortranarray(x0, dtype=np.float64).copy(order="F")
        info = (C.c_int * 3)()
        res = C.c_double()
        if self.o.L.ref_iterative_refine(self.h, _d(F), F.shape[1], _d(X), max_iters, tol, int(transpose), info,
                                         C.byref(res)):
            raise RuntimeError(self.o.err())
        return X, info[0], bool(info[1]), bool(info[2]), res.value

    def solve(self, F, transpose=False):
        F = np.asfortranarray(F, dtype=np.float64)
        X = np.zeros_like(F, order="F")
        sw = (C.c_long * self.p)()
        cc = C.c_long(0)
        if self.o.L.ref_solve(self.h, _d(F), F.shape[1], int(transpose), _d(X), sw, C.byref(cc)):
            raise RuntimeError(self.o.err())
        return X, list(sw), cc.value
