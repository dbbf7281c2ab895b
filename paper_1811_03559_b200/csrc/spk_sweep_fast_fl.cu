// spk_sweep_fast_fl.cu — the sweep launchers of mode SW_FWD_L (tables in
// spk_sweep_launch.cuh; one mode per translation unit for parallel builds).
#include "spk_sweep_launch.cuh"

SPK_SWEEP_LAUNCHERS(fl, SW_FWD_L)
