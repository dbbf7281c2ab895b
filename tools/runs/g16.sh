timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_async.py tests/test_gpu_verify.py -x -q > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
python tools/c3_streams.py > gpurun_out/c3s.log 2>&1
timeout 900 python bench.py --config c5 --no-cpu --no-e2e --steps 3 > gpurun_out/bench_c5.json 2>&1
timeout 900 python bench.py --config c2 --no-cpu --no-e2e --steps 5 > gpurun_out/bench_c2.json 2>&1
