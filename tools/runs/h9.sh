mkdir -p gpurun_out
# solve-sweep time against the column count of one group (compute warps per CTA): --factor-only baseline vs with the forward solve
for r in 64 80 96 112; do
  echo "nrhs=$r factor-only"; timeout 300 python tools/profile_case.py --n 1000000 --k 160 --nrhs $r --reps 3 --prof --factor-only | grep -E "sweep|p="
  echo "nrhs=$r with solve"; timeout 300 python tools/profile_case.py --n 1000000 --k 160 --nrhs $r --reps 3 --prof | grep -E "sweep|p="
done > gpurun_out/h9_tw.log 2>&1
cat gpurun_out/h9_tw.log
