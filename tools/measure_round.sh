set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
CLK=$!
python bench.py --steps 5 --warmup 3 > gpurun_out/fin_bench_c3.json 2> gpurun_out/fin_bench_c3.err
kill $CLK
for c in c1 c2 c4 c5; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/fin_bench_$c.json 2> gpurun_out/fin_bench_$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_bench_c3_ref.json 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-small-k > gpurun_out/fin_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-small-k > /dev/null 2>&1
python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_band_lu_dmma -c 1 -o gpurun_out/fin_prof_lu python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --reps 1 > gpurun_out/fin_ncu_lu.log 2>&1
ls -la gpurun_out | tail -20
