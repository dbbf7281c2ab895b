// spk_sweep_fast_bu.cu — the sweep launchers of mode SW_BWD_U (tables in
// spk_sweep_launch.cuh; one mode per translation unit for parallel builds).
#include "spk_sweep_launch.cuh"

SPK_SWEEP_LAUNCHERS(bu, SW_BWD_U)
