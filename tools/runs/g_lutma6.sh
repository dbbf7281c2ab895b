mkdir -p gpurun_out
( LU_DBG=0 timeout 30 tools/lu_probe 6757 128 2 1; LU_DBG=31 timeout 30 tools/lu_probe 6757 128 2 1 ) > gpurun_out/lu_tma6.log 2>&1
