mkdir -p gpurun_out
for c in c3 c2; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-small-k > gpurun_out/h7_bench_$c.json 2> gpurun_out/h7_bench_$c.err; python - <<PY
import json
d=json.loads(open('gpurun_out/h7_bench_$c.json').read().strip().splitlines()[-1])
print('$c', d['ms_per_step'], d['value'], d.get('backward_error'), {k:v['ms'] for k,v in d['roofline']['classes'].items()})
PY
done
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
tail -3 gpurun_out/gpu_all.log
