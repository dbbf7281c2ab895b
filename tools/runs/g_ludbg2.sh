mkdir -p gpurun_out
( for cfg in "54054 128 148 1 0" "6757 160 148 1 1" "6757 160 148 1 0"; do for dbg in 0 32 64 96; do echo "cfg=$cfg dbg=$dbg: $(LU_DBG=$dbg timeout 30 tools/lu_probe_dbg $cfg | grep 'ms,' | tail -1)"; done; done ) > gpurun_out/lu_dbg2.log 2>&1
