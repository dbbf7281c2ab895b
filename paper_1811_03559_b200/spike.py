"""Python mirror of the reference C++ solver API (``/root/reference/proj/include/spike``).

Same names, argument meaning and error behaviour as the reference, backed by
the sm_100a CUDA library ``libspike_b200.so`` through its C-ABI
(``include/spike_b200.h``).  There is no CPU fallback: importing this module
without the built library, or calling a compute entry point without a GPU,
raises.

Reference symbol                         here
---------------------------------------  -------------------------------------
BandedMatrix (banded_matrix.hpp:14-67)    BandedMatrix (packed (n, ld) array)
DenseBlock   (banded_matrix.hpp:73-91)    numpy 2-D float64 arrays (Fortran order)
PartitionKind/PartitionPlan (partition.hpp:12-37)   same
distribute_threads/compute_ratios/compute_sizes/make_plan (partition.hpp:39-56)  same
FactorOptions, factorize, SpikeFactorization (factorize.hpp:13-77)  same
ReducedLevels, reduce_factorize (factorize.hpp:26-49)  same
SolveStats, solve, transpose_solve, reduced_solve(_transpose), iterative_refine
(solve.hpp:11-51)  same
band_matmul, relative_residual, frobenius_norm, norm1, max_abs (band_ops.hpp)  same
gpu_plan                                 new: arbitrary-p planner for the GPU
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspike_b200.so")

# ----------------------------------------------------------------------------
# errors (the reference's exception types)


class SpikeError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class SingularError(RuntimeError):
    """std::runtime_error: exactly singular column in pivoting mode"""


class DomainError(ValueError):
    """std::domain_error"""


class CudaError(RuntimeError):
    pass


class OutOfRange(IndexError):
    """std::out_of_range"""


class FileFormatError(RuntimeError):
    """std::runtime_error from band_io.cpp (cannot open, bad SPKB magic / dimensions, truncated)."""


_STATUS = {1: InvalidArgument, 2: SingularError, 3: DomainError, 4: CudaError, 5: MemoryError,
           6: CudaError, 7: OutOfRange, 8: FileFormatError}

_lib = None
_lib_lock = threading.Lock()
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class _Plan(C.Structure):
    _fields_ = [("p", C.c_int32), ("bounds", _i64p), ("kinds", _i32p)]


class _Opts(C.Structure):
    _fields_ = [("pivoting", C.c_int32), ("boost_eps", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("partition_full_sweeps", _i64p), ("reduced_coupling_solves", C.c_int64)]


def lib():
    """The loaded CUDA library; raises ImportError when it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1811_03559_b200.build` "
                              "(the GPU path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.spk_last_error.restype = C.c_char_p
        L.spk_version.restype = C.c_char_p
        L.spk_launch_count.restype = C.c_int64
        L.spk_generic_launch_count.restype = C.c_int64
        L.spk_generic_launch_count.argtypes = [C.c_int32]
        L.spk_set_generic_path.argtypes = [C.c_int32]
        L.spk_set_generic_path.restype = None
        L.spk_launch_count.argtypes = [C.c_int32]
        L.spk_compute_ratios.argtypes = [C.c_double, C.c_int32, C.c_int32, _dp, _dp]
        L.spk_compute_ratios.restype = None
        L.spk_distribute_threads.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, C.c_int32, _i32p, _i32p]
        L.spk_compute_sizes.argtypes = [C.c_int64, C.c_int32, _i32p, C.c_double, C.c_double, C.c_int64,
                                        C.c_int64, _i64p]
        L.spk_make_plan.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                    C.c_int32, _i32p, _i64p, _i32p, _i32p, _i32p]
        L.spk_gpu_plan.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                   C.c_int32, _i32p, _i64p, _i32p]
        L.spk_factorize.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                    C.POINTER(_Plan), C.POINTER(_Opts), C.c_void_p,
                                    C.POINTER(C.c_void_p)]
        L.spk_fact_destroy.argtypes = [C.c_void_p]
        L.spk_fact_destroy.restype = None
        L.spk_residual_device.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.POINTER(C.c_double)]
        L.spk_residual_device.restype = C.c_int32
        L.spk_band_norms_device.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                            C.POINTER(C.c_double)]
        L.spk_band_norms_device.restype = C.c_int32
        L.spk_refine.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
                                 C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_void_p, C.POINTER(_RefineC)]
        L.spk_refine.restype = C.c_int32
        L.spk_condest_1norm.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_double)]
        L.spk_condest_1norm.restype = C.c_int32
        L.spk_gpu_plan_ratio.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                         C.c_double, C.c_int32, _i32p, _i64p, _i32p]
        L.spk_gpu_plan_ratio.restype = C.c_int32
        L.spk_calibrate_k.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(_CalibC)]
        L.spk_calibrate_k.restype = C.c_int32
        L.spk_default_k_cache_path.argtypes = [C.c_char_p, C.c_int32]
        L.spk_default_k_cache_path.restype = C.c_int32
        L.spk_write_k_cache.argtypes = [C.c_char_p, C.c_double]
        L.spk_write_k_cache.restype = C.c_int32
        L.spk_read_k_cache.argtypes = [C.c_char_p, C.POINTER(C.c_double), _i32p]
        L.spk_read_k_cache.restype = C.c_int32
        L.spk_spkb_header.argtypes = [C.c_char_p, _i64p, _i32p, _i32p]
        L.spk_spkb_header.restype = C.c_int32
        L.spk_spkb_load.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p]
        L.spk_spkb_load.restype = C.c_int32
        L.spk_spkb_store.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                     C.c_void_p]
        L.spk_spkb_store.restype = C.c_int32
        L.spk_fact_sync.argtypes = [C.c_void_p]
        L.spk_fact_sync.restype = C.c_int32
        L.spk_stream_sync.argtypes = [C.c_void_p]
        L.spk_stream_sync.restype = C.c_int32
        L.spk_fact_info.argtypes = [C.c_void_p, _i64p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p, _i32p]
        L.spk_fact_bounds.argtypes = [C.c_void_p, _i64p]
        L.spk_fact_factor_sweeps.argtypes = [C.c_void_p, _i64p]
        L.spk_fact_tip.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _dp]
        L.spk_fact_level_spike.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, _i32p, _dp]
        L.spk_fact_coupling.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _dp, _i32p, _i32p]
        L.spk_fact_units.argtypes = [C.c_void_p, C.c_int32]
        L.spk_fact_units.restype = C.c_int32
        L.spk_solve.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                C.c_int64, C.c_int32, C.c_void_p, C.POINTER(_Stats)]
        L.spk_reduced_create.argtypes = [_dp, _dp, _dp, _dp, C.c_int32, C.c_int32, C.c_double,
                                         C.POINTER(C.c_void_p)]
        L.spk_reduced_solve.argtypes = [C.c_void_p, C.c_int32, _dp, C.c_int32, _i64p]
        L.spk_reduced_levels.argtypes = [C.c_void_p]
        L.spk_reduced_levels.restype = C.c_int32
        L.spk_reduced_boost_warnings.argtypes = [C.c_void_p]
        L.spk_reduced_boost_warnings.restype = C.c_int32
        L.spk_reduced_destroy.argtypes = [C.c_void_p]
        L.spk_reduced_destroy.restype = None
        L.spk_band_matmul.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                      C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]
        L.spk_generate_band.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_double,
                                        C.c_void_p, C.c_void_p]
        L.spk_generate_rhs.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p]
        L.spk_generate_band_cols.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_double,
                                             C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        L.spk_generate_rhs_rows.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                                            C.c_int64, C.c_void_p]
        # multi-GPU slabs
        L.spk_factorize_slab.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                                         C.POINTER(_Plan), C.POINTER(_Opts), C.c_int32, C.c_int32,
                                         C.c_void_p, C.POINTER(C.c_void_p)]
        L.spk_fact_engine.argtypes = [C.c_void_p]
        L.spk_fact_engine.restype = C.c_int32
        L.spk_fact_open.argtypes = [C.c_void_p]
        L.spk_fact_open.restype = C.c_int32
        L.spk_fact_unit_tips.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.spk_xsolve_exchanges.argtypes = [C.c_void_p, C.c_int32]
        L.spk_xsolve_exchanges.restype = C.c_int32
        L.spk_xsolve_begin.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                       C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.spk_xsolve_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.spk_xsolve_end.argtypes = [C.c_void_p]
        L.spk_xsolve_end.restype = None
        L.spk_reduced_solve_device.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]
        L.spk_reduced_create_device.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_void_p,
                                                C.POINTER(C.c_void_p)]
        # multi-GPU data plane (spk_dist.cu)
        L.spk_comm_unique_id.argtypes = [C.c_void_p]
        L.spk_comm_init.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
        L.spk_comm_wrap.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
        L.spk_comm_destroy.argtypes = [C.c_void_p]
        L.spk_comm_destroy.restype = None
        L.spk_dist_factorize.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.POINTER(_Plan),
                                         C.POINTER(_Opts), C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.spk_dist_solve.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                     C.c_int64, C.c_void_p]
        L.spk_dist_slab.argtypes = [C.c_void_p]
        L.spk_dist_slab.restype = C.c_void_p
        L.spk_dist_destroy.argtypes = [C.c_void_p]
        L.spk_dist_destroy.restype = None
        L.spk_dist_last_error.restype = C.c_char_p
        L.spk_dist_exchange.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_void_p]
        L.spk_arena_cached.restype = C.c_int64
        L.spk_arena_trim.restype = None
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        msg = lib().spk_last_error().decode()
        raise _STATUS.get(rc, SpikeError)(msg)


def _dcheck(rc):
    """Status of a multi-GPU data-plane call (spk_dist.cu keeps its own message)."""
    if rc != 0:
        raise _STATUS.get(rc, SpikeError)(lib().spk_dist_last_error().decode())


def launch_count(reset=False) -> int:
    return int(lib().spk_launch_count(1 if reset else 0))


def fact_engine(fact) -> int:
    """0: general stage programs, 1: small-k engine, 2: small-k with the general hierarchy fallback."""
    return int(lib().spk_fact_engine(fact._h))


def generic_launch_count(reset=False) -> int:
    """Launches of the generic correctness-baseline kernels (0 on tuned shapes)."""
    return int(lib().spk_generic_launch_count(1 if reset else 0))


class generic_path:
    """Context manager: factorizations created inside run every stage on the
    generic kernels (the correctness baseline of the tuned ones)."""

    def __enter__(self):
        lib().spk_set_generic_path(1)
        return self

    def __exit__(self, *exc):
        lib().spk_set_generic_path(0)
        return False


def default_boost_eps() -> float:
    return math.sqrt(np.finfo(np.float64).eps)


# ----------------------------------------------------------------------------
# BandedMatrix / DenseBlock


class BandedMatrix:
    """Packed band, entry (i,j) at data[j, ku+i-j]; data is (n, kl+ku+1) C-order,
    i.e. the reference's column-major (ld, n) layout (banded_matrix.hpp:14-67)."""

    def __init__(self, n: int, kl: int, ku: int, data: Optional[np.ndarray] = None):
        if n < 1:
            raise InvalidArgument("BandedMatrix: n must be >= 1")
        if kl < 0 or ku < 0 or kl >= n or ku >= n:
            raise InvalidArgument("BandedMatrix: need 0 <= kl,ku < n")
        self.n, self.kl, self.ku = int(n), int(kl), int(ku)
        if data is None:
            data = np.zeros((n, kl + ku + 1))
        data = np.ascontiguousarray(data, dtype=np.float64)
        if data.shape != (n, kl + ku + 1):
            raise InvalidArgument("BandedMatrix: data shape mismatch")
        self.data = data

    @staticmethod
    def identity(n: int) -> "BandedMatrix":
        a = BandedMatrix(n, 0, 0)
        a.data[:, 0] = 1.0
        return a

    def ld(self):
        return self.kl + self.ku + 1

    def in_band(self, i, j):
        return 0 <= i < self.n and 0 <= j < self.n and i - j <= self.kl and j - i <= self.ku

    def at(self, i, j):
        if not (0 <= i < self.n and 0 <= j < self.n):
            raise OutOfRange("BandedMatrix::at: index out of range")
        if i - j > self.kl or j - i > self.ku:
            return 0.0
        return float(self.data[j, self.ku + i - j])

    def set(self, i, j, v):
        if not self.in_band(i, j):
            raise OutOfRange("BandedMatrix::set: entry outside the band")
        self.data[j, self.ku + i - j] = v

    def dense(self) -> np.ndarray:
        d = np.zeros((self.n, self.n))
        for j in range(self.n):
            for i in range(max(0, j - self.ku), min(self.n, j + self.kl + 1)):
                d[i, j] = self.data[j, self.ku + i - j]
        return d


def DenseBlock(rows: int, cols: int) -> np.ndarray:
    if rows < 0 or cols < 0:
        raise InvalidArgument("DenseBlock: negative shape")
    return np.zeros((rows, cols), order="F")


def _as_block(f) -> np.ndarray:
    f = np.asarray(f, dtype=np.float64)
    if f.ndim == 1:
        f = f[:, None]
    return np.asfortranarray(f)


# ----------------------------------------------------------------------------
# planning (partition.hpp)


class PartitionKind(enum.IntEnum):
    FirstLast = 0
    InnerSingle = 1
    InnerDual = 2


@dataclass
class PartitionPlan:
    p: int = 1
    bounds: List[int] = field(default_factory=list)
    kinds: List[PartitionKind] = field(default_factory=list)
    threads_used: int = 1
    idle_threads: int = 0
    r12: float = 1.0
    r13: float = 2.0

    def n(self):
        return self.bounds[-1] if self.bounds else 0

    def size(self, i):
        return self.bounds[i + 1] - self.bounds[i]

    def dual_count(self):
        return sum(1 for k in self.kinds if k == PartitionKind.InnerDual)

    def single_count(self):
        return self.p - self.dual_count()


def compute_ratios(k_const: float, n_rhs: int, k: int):
    """(R12, R13) of partition.cpp:47-54."""
    if k_const <= 0.0:
        raise InvalidArgument("compute_ratios: K must be > 0")
    if k < 1:
        raise InvalidArgument("compute_ratios: k must be >= 1")
    if n_rhs < 0:
        raise InvalidArgument("compute_ratios: n_rhs must be >= 0")
    a, b = C.c_double(), C.c_double()
    lib().spk_compute_ratios(k_const, n_rhs, k, C.byref(a), C.byref(b))
    return a.value, b.value


def distribute_threads(t: int, cap_p: int = 0) -> PartitionPlan:
    cap = max(1, 2 * max(t, 1))
    p = C.c_int32()
    kinds = (C.c_int32 * cap)()
    tu, idle = C.c_int32(), C.c_int32()
    _check(lib().spk_distribute_threads(t, cap_p, C.byref(p), kinds, cap, C.byref(tu), C.byref(idle)))
    return PartitionPlan(p=p.value, kinds=[PartitionKind(kinds[i]) for i in range(p.value)],
                         threads_used=tu.value, idle_threads=idle.value)


def compute_sizes(n, skeleton: PartitionPlan, r12, r13, min_single, min_dual):
    p = skeleton.p
    kinds = (C.c_int32 * p)(*[int(k) for k in skeleton.kinds])
    sizes = (C.c_int64 * p)()
    _check(lib().spk_compute_sizes(n, p, kinds, r12, r13, min_single, min_dual, sizes))
    return list(sizes)


def make_plan(n: int, kl: int, ku: int, t: int, r12: float, r13: float) -> PartitionPlan:
    """Reference planner (partition.cpp:89-118): power-of-two p from t threads."""
    cap = max(2, 2 * t + 2)
    p = C.c_int32()
    bounds = (C.c_int64 * (cap + 1))()
    kinds = (C.c_int32 * cap)()
    tu, idle = C.c_int32(), C.c_int32()
    _check(lib().spk_make_plan(n, kl, ku, t, r12, r13, cap, C.byref(p), bounds, kinds, C.byref(tu),
                               C.byref(idle)))
    return PartitionPlan(p=p.value, bounds=list(bounds[:p.value + 1]),
                         kinds=[PartitionKind(kinds[i]) for i in range(p.value)],
                         threads_used=tu.value, idle_threads=idle.value, r12=r12, r13=r13)


def gpu_plan(n: int, kl: int, ku: int, nrhs: int = 1, pivoting: bool = False, p: int = 0,
             r13: Optional[float] = None) -> PartitionPlan:
    """B200 planner: any p >= 1 (not only powers of two), partitions mapped onto SMs;
    equal partitions, or first/last = r13 x inner (the reference's R13) when given."""
    cap = max(4096, 2 * p + 2)
    pp = C.c_int32()
    bounds = (C.c_int64 * (cap + 1))()
    kinds = (C.c_int32 * cap)()
    if r13 is None:
        _check(lib().spk_gpu_plan(n, kl, ku, nrhs, int(pivoting), p, cap, C.byref(pp), bounds, kinds))
    else:
        _check(lib().spk_gpu_plan_ratio(n, kl, ku, nrhs, int(pivoting), p, float(r13), cap, C.byref(pp), bounds,
                                        kinds))
    return PartitionPlan(p=pp.value, bounds=list(bounds[:pp.value + 1]),
                         kinds=[PartitionKind(kinds[i]) for i in range(pp.value)],
                         threads_used=pp.value, idle_threads=0)


# ----------------------------------------------------------------------------
# K calibration (partition.hpp:58-74, partition.cpp:120-170) on the GPU


class _CalibC(C.Structure):
    _fields_ = [("k", C.c_double), ("factor_seconds", C.c_double), ("solve_seconds", C.c_double),
                ("timer_warning", C.c_int32)]


@dataclass
class CalibrationResult:
    k: float = 1.0
    factor_seconds: float = 0.0
    solve_seconds: float = 0.0
    timer_warning: bool = False


def calibrate_k(n_sample: int = 0, k_sample: int = 16, reps: int = 5, stream: int = 0) -> CalibrationResult:
    """K = median t_solve(nrhs = k) / t_factor of one partition, timed on the GPU."""
    out = _CalibC()
    _check(lib().spk_calibrate_k(n_sample, k_sample, reps, stream, C.byref(out)))
    return CalibrationResult(out.k, out.factor_seconds, out.solve_seconds, bool(out.timer_warning))


def default_k_cache_path() -> str:
    buf = C.create_string_buffer(4096)
    _check(lib().spk_default_k_cache_path(buf, 4096))
    return os.fsdecode(buf.value)


def write_k_cache(path, k: float) -> None:
    _check(lib().spk_write_k_cache(os.fsencode(path), float(k)))


def read_k_cache(path) -> Optional[float]:
    v, found = C.c_double(), C.c_int32()
    _check(lib().spk_read_k_cache(os.fsencode(path), C.byref(v), C.byref(found)))
    return float(v.value) if found.value else None


# ----------------------------------------------------------------------------
# factorization (factorize.hpp)


@dataclass
class FactorOptions:
    pivoting: bool = False
    boost_eps: float = field(default_factory=default_boost_eps)


class _Coupling:
    """Factored 2k coupling block of one reduced pair (LUFactors::dense)."""

    def __init__(self, lu: np.ndarray, piv: np.ndarray, fell_back: bool):
        self.lu, self.piv, self.fell_back = lu, piv, fell_back

    def pivoting(self):
        return not self.fell_back

    def uval(self, i, j):
        return float(self.lu[i, j]) if i <= j else 0.0

    def lval(self, i, j):
        if i == j:
            return 1.0
        return float(self.lu[i, j]) if i > j else 0.0


class ReducedLevels:
    """Recursive reduced-system hierarchy (factorize.hpp:26-49), device resident."""

    def __init__(self, owner, handle, p, k, standalone):
        self._owner = owner          # keeps the device object alive
        self._h = handle
        self.p, self.k = p, k
        self._standalone = standalone
        self._v = self._w = self._pairs = None

    def levels(self) -> int:
        if self._standalone:
            return int(lib().spk_reduced_levels(self._h))
        lv = C.c_int32()
        _check(lib().spk_fact_info(self._h, None, None, None, None, None, C.byref(lv), None, None))
        return lv.value

    def unit_rows(self, level):
        return (2 * self.k) << level

    @property
    def boost_warnings(self) -> int:
        if self._standalone:
            return int(lib().spk_reduced_boost_warnings(self._h))
        bw = C.c_int32()
        _check(lib().spk_fact_info(self._h, None, None, None, None, None, None, None, C.byref(bw)))
        return bw.value

    def _spikes(self, which):
        if self._standalone:
            raise SpikeError("spike columns of a standalone reduce_factorize are not mirrored")
        out = []
        for l in range(self.levels()):
            units = lib().spk_fact_units(self._h, l)
            row = []
            for u in range(units):
                h = C.c_int32()
                _check(lib().spk_fact_level_spike(self._h, l, which, u, C.byref(h), None))
                buf = np.zeros(h.value * self.k)
                _check(lib().spk_fact_level_spike(self._h, l, which, u, C.byref(h),
                                                  buf.ctypes.data_as(_dp)))
                row.append(buf.reshape(self.k, h.value).T.copy(order="F"))
            out.append(row)
        return out

    @property
    def v(self):
        if self._v is None:
            self._v = self._spikes(0)
        return self._v

    @property
    def w(self):
        if self._w is None:
            self._w = self._spikes(1)
        return self._w

    @property
    def pairs(self):
        if self._pairs is None:
            if self._standalone:
                raise SpikeError("coupling blocks of a standalone reduce_factorize are not mirrored")
            out = []
            nn = 2 * self.k
            for l in range(self.levels()):
                units = lib().spk_fact_units(self._h, l)
                row = []
                for a in range(units // 2):
                    lu = np.zeros(nn * nn)
                    piv = np.zeros(nn, dtype=np.int32)
                    fb = C.c_int32()
                    _check(lib().spk_fact_coupling(self._h, l, a, lu.ctypes.data_as(_dp),
                                                   piv.ctypes.data_as(_i32p), C.byref(fb)))
                    row.append(_Coupling(lu.reshape(nn, nn).T.copy(), piv, bool(fb.value)))
                out.append(row)
            self._pairs = out
        return self._pairs


class _StandaloneReduced:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            lib().spk_reduced_destroy(self.h)
        except Exception:
            pass


class _FactHandle:
    """Owns one spk_fact*.  Shared by a SpikeFactorization and its
    ReducedLevels without a reference cycle, so dropping the factorization
    frees its HBM immediately (not at the next cycle collection)."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib().spk_fact_destroy(self.h)
                self.h = None
        except Exception:
            pass


class SpikeFactorization:
    """Immutable device-resident SPIKE DS factorization (factorize.hpp:56-74).
    Host mirrors of the tips are fetched on first access."""

    def __init__(self, handle, plan: PartitionPlan, n, kl, ku, options: FactorOptions):
        self._owner = _FactHandle(handle)
        self._h = handle
        self.plan = plan
        self.n, self.kl, self.ku = n, kl, ku
        self.k = max(kl, ku)
        self.options = options
        self._tips = {}
        info = [C.c_int32() for _ in range(3)]
        _check(lib().spk_fact_info(handle, None, None, None, None, None, C.byref(info[0]),
                                   C.byref(info[1]), C.byref(info[2])))
        self.boost_count = info[1].value
        sw = (C.c_int64 * plan.p)()
        _check(lib().spk_fact_factor_sweeps(handle, sw))
        self.factor_sweeps = [int(x) for x in sw]
        self.levels = ReducedLevels(self._owner, handle, plan.p, self.k, standalone=False)

    def p(self):
        return self.plan.p

    def is_dual(self, i):
        return self.plan.kinds[i] == PartitionKind.InnerDual

    def _tipset(self, which):
        if which not in self._tips:
            k = self.k
            out = []
            for i in range(self.plan.p):
                buf = np.zeros(k * k)
                _check(lib().spk_fact_tip(self._h, which, i, buf.ctypes.data_as(_dp)))
                out.append(buf.reshape(k, k).T.copy(order="F"))
            self._tips[which] = out
        return self._tips[which]

    vt = property(lambda self: self._tipset(0))
    vb = property(lambda self: self._tipset(1))
    wt = property(lambda self: self._tipset(2))
    wb = property(lambda self: self._tipset(3))
    bhat = property(lambda self: self._tipset(4))
    chat = property(lambda self: self._tipset(5))


def _plan_struct(plan: PartitionPlan):
    b = np.ascontiguousarray(plan.bounds, dtype=np.int64)
    k = np.ascontiguousarray([int(x) for x in plan.kinds] or [0] * plan.p, dtype=np.int32)
    st = _Plan(plan.p, b.ctypes.data_as(_i64p), k.ctypes.data_as(_i32p))
    return st, (b, k)


def factorize(a: BandedMatrix, plan: PartitionPlan, opts: Optional[FactorOptions] = None,
              stream: int = 0) -> SpikeFactorization:
    """spike::factorize (factorize.hpp:76-77) on the GPU."""
    opts = opts or FactorOptions()
    if plan.n() != a.n:
        raise InvalidArgument("factorize: plan does not match matrix")
    st, keep = _plan_struct(plan)
    o = _Opts(int(bool(opts.pivoting)), float(opts.boost_eps))
    h = C.c_void_p()
    _check(lib().spk_factorize(a.data.ctypes.data, 0, a.n, a.kl, a.ku, C.byref(st), C.byref(o), stream,
                               C.byref(h)))
    fact = SpikeFactorization(h.value, plan, a.n, a.kl, a.ku, opts)
    _check(lib().spk_fact_sync(fact._h))  # factorize() raises like the reference (SingularMatrix)
    return fact


def factorize_device(band_ptr: int, n: int, kl: int, ku: int, plan: PartitionPlan,
                     opts: Optional[FactorOptions] = None, stream: int = 0) -> SpikeFactorization:
    """Factorize a band already resident in HBM (device pointer, (kl+ku+1) x n column-major)."""
    opts = opts or FactorOptions()
    st, keep = _plan_struct(plan)
    o = _Opts(int(bool(opts.pivoting)), float(opts.boost_eps))
    h = C.c_void_p()
    _check(lib().spk_factorize(C.c_void_p(band_ptr), 1, n, kl, ku, C.byref(st), C.byref(o), stream,
                               C.byref(h)))
    fact = SpikeFactorization(h.value, plan, n, kl, ku, opts)
    _check(lib().spk_fact_sync(fact._h))
    return fact


# ----------------------------------------------------------------------------
# solves (solve.hpp)


@dataclass
class SolveStats:
    partition_full_sweeps: List[int] = field(default_factory=list)
    reduced_coupling_solves: int = 0

    def total_full_sweeps(self):
        return sum(self.partition_full_sweeps)


def _solve(fact: SpikeFactorization, f, transpose: bool, stats: Optional[SolveStats]):
    f = _as_block(f)
    if f.shape[0] != fact.n:
        raise InvalidArgument(("transpose_solve" if transpose else "solve") + ": F.rows must equal n")
    nrhs = f.shape[1]
    x = np.zeros((fact.n, nrhs), order="F")
    sw = (C.c_int64 * fact.plan.p)()
    st = _Stats(C.cast(sw, _i64p), 0)
    if nrhs == 0:
        _check(lib().spk_solve(fact._h, int(transpose), None, fact.n, 0, None, fact.n, 0, None, C.byref(st)))
    else:
        _check(lib().spk_solve(fact._h, int(transpose), f.ctypes.data, fact.n, nrhs, x.ctypes.data, fact.n,
                               0, None, C.byref(st)))
        _check(lib().spk_stream_sync(None))  # X is complete once the stream is
    if stats is not None:
        stats.partition_full_sweeps = [int(v) for v in sw]
        stats.reduced_coupling_solves = int(st.reduced_coupling_solves)
    return x


def solve(fact: SpikeFactorization, f, stats: Optional[SolveStats] = None) -> np.ndarray:
    """A X = F on the GPU (solve.hpp:23-24); F is n x nrhs."""
    return _solve(fact, f, False, stats)


def transpose_solve(fact: SpikeFactorization, f, stats: Optional[SolveStats] = None) -> np.ndarray:
    """A^T X = F reusing the same factorization (solve.hpp:28-29)."""
    return _solve(fact, f, True, stats)


def solve_device(fact: SpikeFactorization, f_ptr: int, ldf: int, nrhs: int, x_ptr: int, ldx: int,
                 transpose: bool = False, stream: int = 0) -> None:
    """Device-resident solve: F and X are HBM pointers (column-major)."""
    _check(lib().spk_solve(fact._h, int(transpose), C.c_void_p(f_ptr), ldf, nrhs, C.c_void_p(x_ptr), ldx, 1,
                           stream, None))


def reduce_factorize(vt, vb, wt, wb, p: int, k: int, boost_eps: Optional[float] = None,
                     threads: int = 1) -> ReducedLevels:
    """reduce_factorize (factorize.hpp:45-49); any p >= 1 on the GPU."""
    def pack(blocks):
        arr = np.zeros((p, k, k))
        for i, b in enumerate(blocks[:p]):
            b = np.asarray(b, dtype=np.float64)
            if b.size:
                arr[i] = b.T  # column-major k x k
        return np.ascontiguousarray(arr)
    arrs = [pack(x) for x in (vt, vb, wt, wb)]
    h = C.c_void_p()
    _check(lib().spk_reduced_create(*[a.ctypes.data_as(_dp) for a in arrs], p, k,
                                    boost_eps if boost_eps else default_boost_eps(), C.byref(h)))
    owner = _StandaloneReduced(h.value)
    return ReducedLevels(owner, h.value, p, k, standalone=True)


def _reduced(levels: ReducedLevels, y, transpose, coupling_solves):
    y = _as_block(y)
    if y.shape[0] != 2 * levels.p * levels.k:
        raise InvalidArgument(("reduced_solve_transpose" if transpose else "reduced_solve") +
                              ": tip block has wrong height")
    z = y.copy(order="F")
    cnt = C.c_int64(0)
    if not levels._standalone:
        raise SpikeError("reduced_solve on a factorization's levels: use solve()")
    _check(lib().spk_reduced_solve(levels._h, int(transpose), z.ctypes.data_as(_dp), z.shape[1], C.byref(cnt)))
    if coupling_solves is not None:
        coupling_solves.append(int(cnt.value))
    return z


def reduced_solve(levels: ReducedLevels, ytips, coupling_solves: Optional[list] = None, threads: int = 1):
    return _reduced(levels, ytips, False, coupling_solves)


def reduced_solve_transpose(levels: ReducedLevels, gtips, coupling_solves: Optional[list] = None,
                            threads: int = 1):
    return _reduced(levels, gtips, True, coupling_solves)


# ----------------------------------------------------------------------------
# band ops (band_ops.hpp) on the GPU


def band_matmul(a: BandedMatrix, x, transpose: bool = False) -> np.ndarray:
    x = _as_block(x)
    if x.shape[0] != a.n:
        raise InvalidArgument("band_matmul: X.rows must equal n")
    y = np.zeros_like(x, order="F")
    if x.shape[1]:
        _check(lib().spk_band_matmul(a.data.ctypes.data, a.n, a.kl, a.ku, x.ctypes.data, a.n, x.shape[1],
                                     int(transpose), y.ctypes.data, a.n, 0, None))
    return y


def frobenius_norm(b) -> float:
    return float(np.sqrt(np.sum(np.square(np.asarray(b, dtype=np.float64)))))


def relative_residual(a: BandedMatrix, x, f, transpose: bool = False) -> float:
    """||A X - F||_F / ||F||_F (band_ops.cpp:45-57); A X on the GPU."""
    x, f = _as_block(x), _as_block(f)
    if x.shape[0] != a.n or f.shape[0] != a.n or x.shape[1] != f.shape[1]:
        raise InvalidArgument("relative_residual: inconsistent shapes")
    fn = frobenius_norm(f)
    if fn == 0.0:
        if frobenius_norm(x) == 0.0:
            return 0.0
        raise DomainError("relative_residual: F is zero but X is not")
    r = band_matmul(a, x, transpose) - f
    return frobenius_norm(r) / fn


def norm1(a: BandedMatrix) -> float:
    return float(np.abs(a.data).sum(axis=1).max())


def max_abs(a: BandedMatrix) -> float:
    return float(np.abs(a.data).max())


class _RefineC(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("stagnated", C.c_int32),
                ("residual", C.c_double)]


@dataclass
class RefineResult:
    x: np.ndarray
    iterations: int = 0
    residual: float = 0.0
    converged: bool = False
    stagnated: bool = False


def iterative_refine(fact: SpikeFactorization, a: BandedMatrix, f, x0, max_iters: int, tol: float,
                     transpose: bool = False) -> RefineResult:
    """Residual-correction refinement (solve.cpp:404-432), the whole loop on the
    GPU (spk_refine): residual on the tensor cores, correction solves with the
    factorization, only ||r||_F crossing to the host per iteration."""
    f = _as_block(f)
    x = _as_block(x0).copy(order="F")
    if f.shape != x.shape or f.shape[0] != fact.n or a.n != fact.n:
        raise InvalidArgument("iterative_refine: F.rows must equal n")
    out = _RefineC()
    _check(lib().spk_refine(fact._h, a.data.ctypes.data, f.ctypes.data, fact.n, f.shape[1], x.ctypes.data,
                            fact.n, int(transpose), int(max_iters), float(tol), 0, None, C.byref(out)))
    return RefineResult(x=x, iterations=int(out.iterations), residual=float(out.residual),
                        converged=bool(out.converged), stagnated=bool(out.stagnated))


def refine_device(fact: SpikeFactorization, band_ptr: int, f_ptr: int, ldf: int, nrhs: int, x_ptr: int, ldx: int,
                  max_iters: int, tol: float, transpose: bool = False, stream: int = 0) -> RefineResult:
    """iterative_refine on device buffers: X (x0 on entry) is refined in place."""
    out = _RefineC()
    _check(lib().spk_refine(fact._h, C.c_void_p(band_ptr), C.c_void_p(f_ptr), ldf, nrhs, C.c_void_p(x_ptr), ldx,
                            int(transpose), int(max_iters), float(tol), 1, stream, C.byref(out)))
    return RefineResult(x=None, iterations=int(out.iterations), residual=float(out.residual),
                        converged=bool(out.converged), stagnated=bool(out.stagnated))


# Hager's estimator: the reference's condition_estimate_1norm (src/oracle.cpp:132-166)
def condition_estimate_1norm(fact: SpikeFactorization, a: BandedMatrix) -> float:
    """Hager's kappa_1 estimate (condition_estimate_1norm) with the GPU factorization's solves."""
    cond = C.c_double()
    _check(lib().spk_condest_1norm(fact._h, a.data.ctypes.data, 0, None, C.byref(cond)))
    return float(cond.value)


def condition_estimate_device(fact: SpikeFactorization, band_ptr: int, stream: int = 0) -> float:
    cond = C.c_double()
    _check(lib().spk_condest_1norm(fact._h, C.c_void_p(band_ptr), 1, stream, C.byref(cond)))
    return float(cond.value)


def residual_device(band_ptr: int, n: int, kl: int, ku: int, x_ptr: int, ldx: int, f_ptr: int, ldf: int,
                    ncols: int, transpose: bool = False, r_ptr: int = 0, ldr: int = 0, stream: int = 0) -> np.ndarray:
    """R = F - op(A) X on device buffers; returns per column
    [||r||_2^2, ||f||_2^2, max|r|, max|x|] (ncols x 4)."""
    out = np.zeros((max(ncols, 1), 4))
    _check(lib().spk_residual_device(C.c_void_p(band_ptr), n, kl, ku, C.c_void_p(x_ptr), ldx, C.c_void_p(f_ptr),
                                     ldf, ncols, int(transpose), C.c_void_p(r_ptr or None), ldr or n, stream,
                                     out.ctypes.data_as(C.POINTER(C.c_double))))
    return out[:ncols]


def band_norms_device(band_ptr: int, n: int, kl: int, ku: int, stream: int = 0):
    """(||A||_1, ||A||_inf, max|a_ij|) of a device band."""
    out = (C.c_double * 3)()
    _check(lib().spk_band_norms_device(C.c_void_p(band_ptr), n, kl, ku, stream, out))
    return float(out[0]), float(out[1]), float(out[2])


def backward_error_device(band_ptr: int, n: int, kl: int, ku: int, x_ptr: int, ldx: int, f_ptr: int, ldf: int,
                          ncols: int, transpose: bool = False, stream: int = 0) -> float:
    """Normwise backward error max_c ||r_c||_inf / (||op(A)||_inf ||x_c||_inf)."""
    st = residual_device(band_ptr, n, kl, ku, x_ptr, ldx, f_ptr, ldf, ncols, transpose, stream=stream)
    n1, ninf, _ = band_norms_device(band_ptr, n, kl, ku, stream)
    an = n1 if transpose else ninf
    return float(max((r[2] / (an * r[3]) if r[3] > 0 else (0.0 if r[2] == 0 else math.inf)) for r in st)) if ncols else 0.0


# ----------------------------------------------------------------------------
# .spkb band files (band_io.hpp / band_io.cpp:98-143)


def _path(p) -> bytes:
    return os.fsencode(p)


def spkb_header(path):
    """(n, kl, ku) of a .spkb file."""
    n, kl, ku = C.c_int64(), C.c_int32(), C.c_int32()
    _check(lib().spk_spkb_header(_path(path), C.byref(n), C.byref(kl), C.byref(ku)))
    return int(n.value), int(kl.value), int(ku.value)


def read_spkb(path) -> BandedMatrix:
    """read_matrix on a .spkb file (band_io.cpp:98-110, :145-155)."""
    n, kl, ku = spkb_header(path)
    data = np.zeros((n, kl + ku + 1))
    _check(lib().spk_spkb_load(_path(path), 0, n, data.ctypes.data, 0, None))
    return BandedMatrix(n, kl, ku, data)


def read_matrix(path) -> BandedMatrix:
    """band_io.cpp:145-155 for the binary format (MatrixMarket text is out of scope)."""
    with open(path, "rb") as fh:
        head = fh.read(4)
    if not head:
        raise FileFormatError("empty matrix file")
    if head != b"SPKB":
        raise FileFormatError("MatrixMarket input is not supported; convert to .spkb")
    return read_spkb(path)


def write_spkb(a: BandedMatrix, path) -> None:
    """write_matrix(a, path, MatrixFormat::Spkb) (band_io.cpp:114-122)."""
    _check(lib().spk_spkb_store(_path(path), a.data.ctypes.data, a.n, a.kl, a.ku, 0, None))


def load_spkb_device(path, dst_ptr: int, col0: int = 0, ncols: Optional[int] = None, stream: int = 0):
    """Columns [col0, col0+ncols) of a .spkb band straight into HBM (a slab's
    window with its halo columns); returns (n, kl, ku) of the file."""
    n, kl, ku = spkb_header(path)
    ncols = n - col0 if ncols is None else ncols
    _check(lib().spk_spkb_load(_path(path), col0, ncols, C.c_void_p(dst_ptr), 1, stream))
    return n, kl, ku


def store_spkb_device(path, band_ptr: int, n: int, kl: int, ku: int, stream: int = 0) -> None:
    _check(lib().spk_spkb_store(_path(path), C.c_void_p(band_ptr), n, kl, ku, 1, stream))


# ----------------------------------------------------------------------------
# device-side input generation (include/spike_b200_gen.h)


def generate_band_device(seed: int, n: int, kl: int, ku: int, dd: float, band_ptr: int, stream: int = 0):
    _check(lib().spk_generate_band(seed, n, kl, ku, dd, C.c_void_p(band_ptr), stream))


def generate_rhs_device(seed: int, n: int, ncols: int, f_ptr: int, ldf: int, stream: int = 0):
    _check(lib().spk_generate_rhs(seed, n, ncols, C.c_void_p(f_ptr), ldf, stream))
