mkdir -p gpurun_out
( for cfg in "54054 128 148 1 0" "6757 160 148 1 1" "6757 160 148 1 0" "6757 160 148 0 1"; do echo "plain $cfg: $(timeout 30 tools/lu_probe_plain $cfg | grep 'ms,' | tail -1)"; for dbg in 32 96; do echo "cfg=$cfg dbg=$dbg: $(LU_DBG=$dbg timeout 30 tools/lu_probe_dbg $cfg | grep 'ms,' | tail -1)"; done; done ) > gpurun_out/lu3.log 2>&1
