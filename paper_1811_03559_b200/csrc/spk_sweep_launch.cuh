// spk_sweep_launch.cuh — launch tables of the sweep kernels, one set per mode.
//
// Each spk_sweep_fast_<mode>.cu includes this header and instantiates the
// three launchers of one sweep mode with SPK_SWEEP_LAUNCHERS (the modes are
// split across translation units so nvcc builds the templates in parallel).
// The tables are built by fold expressions over the template parameters the
// dispatcher (spk_capi.cu, Exec::run_fast_sweep) can ask for:
//   k_sweep_fast   TR in 1..8 (32-row register tiles), NC in {1, 2, 4}, PIV (FWD_L only)
//   k_sweep_dmma   NTW in {3, 5, 9, 13, 17, 21, 25}, PAIR for NTW >= 9
//   k_sweep_dmma2  NTW in {3, 5, 9, 13, 17, 21, 25}, PAIR
#pragma once

#include "spk_launch.h"
#include "spk_sweep_dmma.cuh"
#include "spk_sweep_dmma2.cuh"
#include "spk_sweep_fast.cuh"

#include <cuda_runtime.h>

#include <utility>

namespace spk {

using SweepFn = void (*)(FastSweepArgs);

template <int MODE, bool PIV, int TR>
SweepFn pick_fast_nc(int nc) {
    if (nc == 1) return k_sweep_fast<TR, 1, MODE, PIV>;
    if (nc == 2) return k_sweep_fast<TR, 2, MODE, PIV>;
    if (nc == 4) return k_sweep_fast<TR, 4, MODE, PIV>;
    return nullptr;
}

template <int MODE, bool PIV, int... TR>
SweepFn pick_fast(int tr, int nc, std::integer_sequence<int, TR...>) {
    SweepFn fn = nullptr;
    ((tr == TR ? (void)(fn = pick_fast_nc<MODE, PIV, TR>(nc)) : (void)0), ...);
    return fn;
}

using NtwList = std::integer_sequence<int, 3, 5, 9, 13, 17, 21, 25>;

template <int MODE, int... NTW>
SweepFn pick_dmma(int ntw, bool pair, std::integer_sequence<int, NTW...>) {
    SweepFn fn = nullptr;
    if (pair)  // the window split over a warp pair needs >= 9 tiles
        ((ntw == NTW && NTW >= 9 ? (void)(fn = k_sweep_dmma<(NTW >= 9 ? NTW : 9), MODE, true>) : (void)0), ...);
    else
        ((ntw == NTW ? (void)(fn = k_sweep_dmma<NTW, MODE>) : (void)0), ...);
    return fn;
}

template <int MODE, int... NTW>
SweepFn pick_dmma2(int ntw, bool pair, std::integer_sequence<int, NTW...>) {
    SweepFn fn = nullptr;
    if (pair)
        ((ntw == NTW ? (void)(fn = k_sweep_dmma2<NTW, MODE, true>) : (void)0), ...);
    else
        ((ntw == NTW ? (void)(fn = k_sweep_dmma2<NTW, MODE>) : (void)0), ...);
    return fn;
}

template <int MODE>
bool launch_fast_mode(int tr, int nc, bool piv, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A,
                      cudaStream_t s) {
    SweepFn fn = nullptr;
    if (piv && MODE == SW_FWD_L)
        fn = pick_fast<MODE, true>(tr, nc, std::integer_sequence<int, 1, 2, 3, 4, 5, 6, 7, 8>{});
    else if (!piv)
        fn = pick_fast<MODE, false>(tr, nc, std::integer_sequence<int, 1, 2, 3, 4, 5, 6, 7, 8>{});
    if (!fn) return false;
    set_smem_attr((const void*)fn, 227 * 1024);
    fn<<<grid, 32 * nwarps, smem, s>>>(A);
    count_launch();
    return true;
}

template <int MODE>
bool launch_dmma_mode(int ntw, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A, cudaStream_t s,
                      bool pair) {
    SweepFn fn = pick_dmma<MODE>(ntw, pair, NtwList{});
    if (!fn) return false;
    set_smem_attr((const void*)fn, 227 * 1024);
    fn<<<grid, 32 * nwarps, smem, s>>>(A);
    count_launch();
    return true;
}

template <int MODE>
bool launch_dmma2_mode(int ntw, int ncw, dim3 grid, const FastSweepArgs& A, cudaStream_t s, bool pair) {
    SweepFn fn = pick_dmma2<MODE>(ntw, pair, NtwList{});
    if (!fn) return false;
    const size_t smem = dmma2_sweep_smem(ntw, ncw, pair);
    if (smem > 227 * 1024) return false;
    set_smem_attr((const void*)fn, 227 * 1024);
    fn<<<grid, 32 * (ncw + kDmma2Producers), smem, s>>>(A);
    count_launch();
    return true;
}

}  // namespace spk

// the three C++ launchers of one mode (declared in spk_launch.h)
#define SPK_SWEEP_LAUNCHERS(suffix, MODE)                                                                       \
    namespace spk {                                                                                             \
    bool launch_sweep_fast_##suffix(int tr, int nc, bool piv, int nwarps, dim3 grid, size_t smem,               \
                                    const FastSweepArgs& A, cudaStream_t s) {                                   \
        return launch_fast_mode<MODE>(tr, nc, piv, nwarps, grid, smem, A, s);                                   \
    }                                                                                                           \
    bool launch_sweep_dmma_##suffix(int ntw, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A,        \
                                    cudaStream_t s, bool pair) {                                                \
        return launch_dmma_mode<MODE>(ntw, nwarps, grid, smem, A, s, pair);                                     \
    }                                                                                                           \
    bool launch_sweep_dmma2_##suffix(int ntw, int ncw, dim3 grid, const FastSweepArgs& A, cudaStream_t s,       \
                                     bool pair) {                                                               \
        return launch_dmma2_mode<MODE>(ntw, ncw, grid, A, s, pair);                                             \
    }                                                                                                           \
    }
