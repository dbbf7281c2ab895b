mkdir -p gpurun_out
( for np in 2 1 3 4; do
  echo "nprod=$np nrhs=80"; SPK_NPROD=$np timeout 300 python tools/profile_case.py --n 1000000 --k 160 --nrhs 80 --reps 3 --prof | grep -E "sweep|band_lu"
done
for np in 2 1; do echo "nprod=$np nrhs=96";  SPK_NPROD=$np timeout 300 python tools/profile_case.py --n 1000000 --k 160 --nrhs 96 --reps 3 --prof | grep -E "sweep"; done
echo "C3"; timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e --no-small-k | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('c3', d['ms_per_step'], d['value'], d.get('backward_error'), {k:v['ms'] for k,v in d['roofline']['classes'].items()})"
echo "C5"; timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-small-k | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('c5', d['ms_per_step'], d['value'], d.get('backward_error'), {k:v['ms'] for k,v in d['roofline']['classes'].items()})"
) > gpurun_out/h10.log 2>&1
cat gpurun_out/h10.log
