python tools/profile_case.py --n 2000000 --k 128 --nrhs 32 --reps 1 --factor-only > gpurun_out/plain_lu5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_band_lu_dmma -c 1 -o gpurun_out/prof_lu5 python tools/profile_case.py --n 2000000 --k 128 --nrhs 32 --reps 1 --factor-only > gpurun_out/ncu_lu5.log 2>&1
echo done
