mkdir -p gpurun_out
( for np in 2 3 4 6; do
  echo "nprod=$np nrhs=80"; SPK_NPROD=$np timeout 300 python tools/profile_case.py --n 1000000 --k 160 --nrhs 80 --reps 3 --prof | grep -E "sweep"
done
for np in 2 3 4; do echo "nprod=$np nrhs=160";  SPK_NPROD=$np timeout 300 python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 3 --prof | grep -E "sweep"; done
) > gpurun_out/h11.log 2>&1
cat gpurun_out/h11.log
