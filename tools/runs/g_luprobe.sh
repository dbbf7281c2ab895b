set -x
mkdir -p gpurun_out
( tools/lu_probe_plain 6757 160 148; tools/lu_probe 6757 160 148; tools/lu_probe 6757 160 1; tools/lu_probe 54054 128 1 ) > gpurun_out/lu_probe.log 2>&1
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
