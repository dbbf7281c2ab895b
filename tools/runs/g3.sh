timeout 600 python -m pytest tests/test_gpu_smallk.py -x -q > gpurun_out/smallk.log 2>&1; echo smallk rc=$? >> gpurun_out/smallk.log
timeout 120 python tools/sk_probe.py > gpurun_out/sk_probe.log 2>&1
timeout 120 python tools/sk_probe.py 1024 >> gpurun_out/sk_probe.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
tail -n 3 gpurun_out/smallk.log gpurun_out/gpu_all.log
