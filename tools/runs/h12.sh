mkdir -p gpurun_out
( for np in 2 3 1; do echo "nprod=$np C3"; SPK_NPROD=$np timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e --no-small-k | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('c3', d['ms_per_step'], d['value'], d.get('backward_error'), {k:v['ms'] for k,v in d['roofline']['classes'].items()})"
done
echo "C2"; timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e --no-small-k | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('c2', d['ms_per_step'], d['value'], d.get('backward_error'), {k:v['ms'] for k,v in d['roofline']['classes'].items()})"
) > gpurun_out/h12.log 2>&1
cat gpurun_out/h12.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
tail -3 gpurun_out/gpu_all.log
