mkdir -p gpurun_out
( for cfg in "6757 160 148 1" "54054 128 148 1"; do echo "plain $cfg: $(timeout 30 tools/lu_probe_plain $cfg | grep 'ms,' | tail -1)"; for dbg in 32 96; do echo "cfg=$cfg dbg=$dbg: $(LU_DBG=$dbg timeout 30 tools/lu_probe_dbg $cfg | grep 'ms,' | tail -1)"; done; done ) > gpurun_out/lu_out.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_scale_parity.py -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
