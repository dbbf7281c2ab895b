// spk_sweep_fast_fut.cu — the sweep launchers of mode SW_FWD_UT (tables in
// spk_sweep_launch.cuh; one mode per translation unit for parallel builds).
#include "spk_sweep_launch.cuh"

SPK_SWEEP_LAUNCHERS(fut, SW_FWD_UT)
