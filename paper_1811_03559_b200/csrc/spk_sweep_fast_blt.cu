// spk_sweep_fast_blt.cu — the sweep launchers of mode SW_BWD_LT (tables in
// spk_sweep_launch.cuh; one mode per translation unit for parallel builds).
#include "spk_sweep_launch.cuh"

SPK_SWEEP_LAUNCHERS(blt, SW_BWD_LT)
