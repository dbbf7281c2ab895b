# TMA-staged DMMA LU: phase probe (TMA on / element path), then the GPU suite
set -x
mkdir -p gpurun_out
( timeout 60 tools/lu_probe_plain 6757 160 148 1; timeout 60 tools/lu_probe_plain 6757 160 148 0; timeout 60 tools/lu_probe 6757 160 148 1; timeout 60 tools/lu_probe 54054 128 1 1; timeout 60 tools/lu_probe_plain 54054 128 296 1; timeout 60 tools/lu_probe_plain 54054 128 296 0 ) > gpurun_out/lu_tma.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -5 gpurun_out/gpu_tests.log
