// spk_sweep_fast_fut.cu — instantiations of the sweep kernels for SW_FWD_UT
// (register-window DFMA: k_sweep_fast; blocked DMMA: k_sweep_dmma).
// Split per mode so nvcc builds the templates in parallel.
#include "spk_sweep_fast.cuh"
#include "spk_sweep_dmma.cuh"
#include "spk_sweep_dmma2.cuh"
#include "spk_launch.h"

#include <cuda_runtime.h>

namespace spk {

bool launch_sweep_fast_fut(int tr, int nc, bool piv, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A, cudaStream_t s) {
    void (*fn)(FastSweepArgs) = nullptr;
    if (tr == 1 && nc == 1 && piv == false) fn = k_sweep_fast<1, 1, SW_FWD_UT, false>;
    if (tr == 1 && nc == 2 && piv == false) fn = k_sweep_fast<1, 2, SW_FWD_UT, false>;
    if (tr == 1 && nc == 4 && piv == false) fn = k_sweep_fast<1, 4, SW_FWD_UT, false>;
    if (tr == 2 && nc == 1 && piv == false) fn = k_sweep_fast<2, 1, SW_FWD_UT, false>;
    if (tr == 2 && nc == 2 && piv == false) fn = k_sweep_fast<2, 2, SW_FWD_UT, false>;
    if (tr == 2 && nc == 4 && piv == false) fn = k_sweep_fast<2, 4, SW_FWD_UT, false>;
    if (tr == 3 && nc == 1 && piv == false) fn = k_sweep_fast<3, 1, SW_FWD_UT, false>;
    if (tr == 3 && nc == 2 && piv == false) fn = k_sweep_fast<3, 2, SW_FWD_UT, false>;
    if (tr == 3 && nc == 4 && piv == false) fn = k_sweep_fast<3, 4, SW_FWD_UT, false>;
    if (tr == 4 && nc == 1 && piv == false) fn = k_sweep_fast<4, 1, SW_FWD_UT, false>;
    if (tr == 4 && nc == 2 && piv == false) fn = k_sweep_fast<4, 2, SW_FWD_UT, false>;
    if (tr == 4 && nc == 4 && piv == false) fn = k_sweep_fast<4, 4, SW_FWD_UT, false>;
    if (tr == 5 && nc == 1 && piv == false) fn = k_sweep_fast<5, 1, SW_FWD_UT, false>;
    if (tr == 5 && nc == 2 && piv == false) fn = k_sweep_fast<5, 2, SW_FWD_UT, false>;
    if (tr == 5 && nc == 4 && piv == false) fn = k_sweep_fast<5, 4, SW_FWD_UT, false>;
    if (tr == 6 && nc == 1 && piv == false) fn = k_sweep_fast<6, 1, SW_FWD_UT, false>;
    if (tr == 6 && nc == 2 && piv == false) fn = k_sweep_fast<6, 2, SW_FWD_UT, false>;
    if (tr == 6 && nc == 4 && piv == false) fn = k_sweep_fast<6, 4, SW_FWD_UT, false>;
    if (tr == 7 && nc == 1 && piv == false) fn = k_sweep_fast<7, 1, SW_FWD_UT, false>;
    if (tr == 7 && nc == 2 && piv == false) fn = k_sweep_fast<7, 2, SW_FWD_UT, false>;
    if (tr == 7 && nc == 4 && piv == false) fn = k_sweep_fast<7, 4, SW_FWD_UT, false>;
    if (tr == 8 && nc == 1 && piv == false) fn = k_sweep_fast<8, 1, SW_FWD_UT, false>;
    if (tr == 8 && nc == 2 && piv == false) fn = k_sweep_fast<8, 2, SW_FWD_UT, false>;
    if (tr == 8 && nc == 4 && piv == false) fn = k_sweep_fast<8, 4, SW_FWD_UT, false>;
    if (!fn) return false;
    static bool attr_done[2][9][5] = {};
    if (!attr_done[piv][tr][nc]) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr_done[piv][tr][nc] = true;
    }
    fn<<<grid, 32 * nwarps, smem, s>>>(A);
    count_launch();
    return true;
}

bool launch_sweep_dmma_fut(int ntw, int nwarps, dim3 grid, size_t smem, const FastSweepArgs& A, cudaStream_t s,
                          bool pair) {
    void (*fn)(FastSweepArgs) = nullptr;
    int slot = -1;
    if (!pair) {
        if (ntw == 3) { fn = k_sweep_dmma<3, SW_FWD_UT>; slot = 0; }
        if (ntw == 5) { fn = k_sweep_dmma<5, SW_FWD_UT>; slot = 1; }
        if (ntw == 9) { fn = k_sweep_dmma<9, SW_FWD_UT>; slot = 2; }
        if (ntw == 13) { fn = k_sweep_dmma<13, SW_FWD_UT>; slot = 3; }
        if (ntw == 17) { fn = k_sweep_dmma<17, SW_FWD_UT>; slot = 4; }
        if (ntw == 21) { fn = k_sweep_dmma<21, SW_FWD_UT>; slot = 5; }
        if (ntw == 25) { fn = k_sweep_dmma<25, SW_FWD_UT>; slot = 6; }
    } else {
        if (ntw == 9) { fn = k_sweep_dmma<9, SW_FWD_UT, true>; slot = 7; }
        if (ntw == 13) { fn = k_sweep_dmma<13, SW_FWD_UT, true>; slot = 8; }
        if (ntw == 17) { fn = k_sweep_dmma<17, SW_FWD_UT, true>; slot = 9; }
        if (ntw == 21) { fn = k_sweep_dmma<21, SW_FWD_UT, true>; slot = 10; }
        if (ntw == 25) { fn = k_sweep_dmma<25, SW_FWD_UT, true>; slot = 11; }
    }
    if (!fn) return false;
    static bool attr_done[12] = {};
    if (!attr_done[slot]) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr_done[slot] = true;
    }
    fn<<<grid, 32 * nwarps, smem, s>>>(A);
    count_launch();
    return true;
}

bool launch_sweep_dmma2_fut(int ntw, int ncw, dim3 grid, const FastSweepArgs& A, cudaStream_t s, bool pair) {
    void (*fn)(FastSweepArgs) = nullptr;
    int slot = -1;
    if (!pair) {
        if (ntw == 3) { fn = k_sweep_dmma2<3, SW_FWD_UT>; slot = 0; }
        if (ntw == 5) { fn = k_sweep_dmma2<5, SW_FWD_UT>; slot = 1; }
        if (ntw == 9) { fn = k_sweep_dmma2<9, SW_FWD_UT>; slot = 2; }
        if (ntw == 13) { fn = k_sweep_dmma2<13, SW_FWD_UT>; slot = 3; }
        if (ntw == 17) { fn = k_sweep_dmma2<17, SW_FWD_UT>; slot = 4; }
        if (ntw == 21) { fn = k_sweep_dmma2<21, SW_FWD_UT>; slot = 5; }
        if (ntw == 25) { fn = k_sweep_dmma2<25, SW_FWD_UT>; slot = 6; }
    } else {
        if (ntw == 3) { fn = k_sweep_dmma2<3, SW_FWD_UT, true>; slot = 13; }
        if (ntw == 5) { fn = k_sweep_dmma2<5, SW_FWD_UT, true>; slot = 7; }
        if (ntw == 9) { fn = k_sweep_dmma2<9, SW_FWD_UT, true>; slot = 8; }
        if (ntw == 13) { fn = k_sweep_dmma2<13, SW_FWD_UT, true>; slot = 9; }
        if (ntw == 17) { fn = k_sweep_dmma2<17, SW_FWD_UT, true>; slot = 10; }
        if (ntw == 21) { fn = k_sweep_dmma2<21, SW_FWD_UT, true>; slot = 11; }
        if (ntw == 25) { fn = k_sweep_dmma2<25, SW_FWD_UT, true>; slot = 12; }
    }
    if (!fn) return false;
    const size_t smem = dmma2_sweep_smem(ntw, ncw, pair);
    if (smem > 227 * 1024) return false;
    static bool attr_done[14] = {};
    if (!attr_done[slot]) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr_done[slot] = true;
    }
    fn<<<grid, 32 * (ncw + kDmma2Producers), smem, s>>>(A);
    count_launch();
    return true;
}

}  // namespace spk
