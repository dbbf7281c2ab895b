mkdir -p gpurun_out
( for cfg in "6757 128 4 1" "6757 128 4 0" "6757 128 1 1" "6757 160 148 1" "6757 160 148 0"; do
   for dbg in 0 31; do echo "cfg=$cfg dbg=$dbg: $(LU_DBG=$dbg timeout 30 tools/lu_probe $cfg | grep 'ms,' | tail -1)"; done; done ) > gpurun_out/lu_tma5.log 2>&1
