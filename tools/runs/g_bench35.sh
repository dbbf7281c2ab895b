mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config c5 --no-cpu --steps 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
