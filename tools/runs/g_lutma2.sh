set -x
mkdir -p gpurun_out
for k in 40 64 96 128 160; do for dbg in 0 1 2 3 4; do echo "k=$k dbg=$dbg"; LU_DBG=$dbg timeout 30 tools/lu_probe 6757 $k 4 1 | grep "ms,"; done; done > gpurun_out/lu_tma2.log 2>&1
