mkdir -p gpurun_out
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e --no-small-k > gpurun_out/h4_bench_c3.json 2> gpurun_out/h4_bench_c3.err; python - <<PY
import json
d=json.loads(open('gpurun_out/h4_bench_c3.json').read().strip().splitlines()[-1])
print('c3', d['ms_per_step'], d['value'], d.get('backward_error'), {k:v['ms'] for k,v in d['roofline']['classes'].items()})
PY
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
tail -3 gpurun_out/gpu_all.log
