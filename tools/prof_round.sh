set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks.csv &
CLK=$!
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_full.json 2> gpurun_out/bench_c3_full.err
kill $CLK
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c3_ref.json 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_dmma2 -s 2 -c 3 -o gpurun_out/prof_sweep python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_band_lu -c 1 -o gpurun_out/prof_lu python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --reps 1 > gpurun_out/ncu_full_lu.log 2>&1
ls -la gpurun_out
