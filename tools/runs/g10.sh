python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --reps 1 > gpurun_out/plain_lu.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_band_lu_dmma -c 1 -o gpurun_out/prof_lu python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --reps 1 > gpurun_out/ncu_lu.log 2>&1
echo done
