set -x
mkdir -p gpurun_out
( LU_DBG=3 timeout 120 compute-sanitizer --tool memcheck --show-backtrace device tools/lu_probe 6757 128 1 1 2>&1 | head -60
  timeout 30 tools/lu_probe 54054 128 1 1 | grep "ms,"
  timeout 30 tools/lu_probe 6760 128 1 1 | grep "ms,"
  timeout 30 tools/lu_probe 6757 128 1 1 | grep "ms,"
  timeout 30 tools/lu_probe 20000 128 1 1 | grep "ms,"
  timeout 30 tools/lu_probe 54054 160 1 1 | grep "ms," ) > gpurun_out/lu_tma3.log 2>&1
