mkdir -p gpurun_out
( for c in c5 c2 c4 c3; do
  timeout 900 python bench.py --config $c --steps 4 --warmup 3 --no-cpu --no-e2e --no-small-k | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', d['ms_per_step'], d['value'], d.get('backward_error'), {k:v['ms'] for k,v in d['roofline']['classes'].items()})"
done ) > gpurun_out/h18.log 2>&1
cat gpurun_out/h18.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all_h18.log 2>&1; echo rc=$? >> gpurun_out/gpu_all_h18.log
tail -3 gpurun_out/gpu_all_h18.log
