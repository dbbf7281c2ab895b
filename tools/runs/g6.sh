timeout 600 python -m pytest tests/test_gpu_smallk.py -x -q > gpurun_out/smallk.log 2>&1; echo smallk rc=$? >> gpurun_out/smallk.log
for p in 0 592 2048; do timeout 120 python tools/sk_probe.py $p > gpurun_out/sk_probe_$p.log 2>&1; done
timeout 300 python tools/sk_probe.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sk_launches.csv python tools/sk_probe.py > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
