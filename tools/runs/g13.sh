python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --reps 1 > gpurun_out/plain_sw.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_dmma2 -s 2 -c 1 -o gpurun_out/prof_sweep python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --reps 1 > gpurun_out/ncu_sw.log 2>&1
echo done
