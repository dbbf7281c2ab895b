mkdir -p gpurun_out
( for e in 0 1; do for c in c5 c2; do
  if [ $e = 1 ]; then export SPK_DMMA2_ALWAYS=1; else unset SPK_DMMA2_ALWAYS; fi
  echo "always=$e $c"; timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e --no-small-k | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', d['ms_per_step'], d['value'], d.get('backward_error'), {k:v['ms'] for k,v in d['roofline']['classes'].items()})"
done; done ) > gpurun_out/h14.log 2>&1
cat gpurun_out/h14.log
