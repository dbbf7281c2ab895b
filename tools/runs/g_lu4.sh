mkdir -p gpurun_out
( for cfg in "54054 128 148 1 0" "54054 128 148 1 1" "6757 160 148 1 1" "6757 160 148 1 0"; do for b in lu_probe_v1 lu_probe_plain lu_probe_v3; do echo "$b $cfg: $(timeout 30 tools/$b $cfg | grep 'ms,' | tail -1 | cut -c1-60)"; done; done ) > gpurun_out/lu4.log 2>&1
