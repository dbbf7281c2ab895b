mkdir -p gpurun_out
( for cfg in "6757 160 148 1" "54054 128 148 1"; do for dbg in 0 32 64 96; do echo "cfg=$cfg dbg=$dbg: $(LU_DBG=$dbg timeout 30 tools/lu_probe_dbg $cfg | grep 'ms,' | tail -1)"; done; done ) > gpurun_out/lu_dbg.log 2>&1
