mkdir -p gpurun_out
( for cfg in "6757 128 4 1" "6757 128 2 1" "6757 128 3 1" "54054 128 4 1" "6757 128 4 0" "20000 128 8 1" "54054 128 8 1" "54054 128 16 1"; do
   for dbg in 0 3 7 15 31; do echo "cfg=$cfg dbg=$dbg: $(LU_DBG=$dbg timeout 30 tools/lu_probe $cfg | grep 'ms,' | tail -1)"; done; done ) > gpurun_out/lu_tma4.log 2>&1
