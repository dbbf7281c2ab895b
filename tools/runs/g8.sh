timeout 600 python -m pytest tests/test_gpu_smallk.py -x -q > gpurun_out/smallk.log 2>&1; echo smallk rc=$? >> gpurun_out/smallk.log
python tools/sk_check.py > gpurun_out/skc.log 2>&1
python tools/sk_trace.py > gpurun_out/trace.log 2>&1
python tools/sk_probe.py > gpurun_out/sk_probe.log 2>&1
