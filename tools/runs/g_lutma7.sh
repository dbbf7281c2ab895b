mkdir -p gpurun_out
( for cfg in "6757 128 4 1" "6757 160 148 1" "6757 160 148 0" "54054 128 296 1" "54054 128 296 0"; do echo "cfg=$cfg: $(timeout 30 tools/lu_probe_plain $cfg | grep 'ms,' | tail -1)"; done
  timeout 30 tools/lu_probe 6757 160 148 1 ) > gpurun_out/lu_tma7.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
