mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
tail -3 gpurun_out/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/h1_bench_c3.json 2> gpurun_out/h1_bench_c3.err
tail -c 3000 gpurun_out/h1_bench_c3.json
