timeout 600 python -m pytest tests/test_gpu_smallk.py -x -q > gpurun_out/smallk.log 2>&1; echo smallk rc=$? >> gpurun_out/smallk.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
