# Round-end measurements (one gpurun call): bench lines for C1..C5 and the
# reference arm, the C3 launch list, and ncu --set full captures of the top
# kernels (each only after its own command exited 0 without ncu).
set -x
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > $O/clocks.csv &
CLK=$!
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
kill $CLK
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_c3_reference.json 2> $O/bench_c3_reference.err
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
for c in c2 c4 c5; do timeout 900 python bench.py --config $c --no-cpu --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; done
# C3 launch list (cold-cache, serialised: shares, not absolutes)
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-small-k > $O/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-small-k > $O/ncu_launch.log 2>&1
# C1 launch list
timeout 300 python tools/sk_probe.py > $O/plain_c1.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c1_launches.csv python tools/sk_probe.py > $O/ncu_c1_launch.log 2>&1
# top kernels
timeout 600 python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1 > $O/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep_dmma2 -s 2 -c 2 -o $O/prof_sweep python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1 > $O/ncu_sweep.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_band_lu_dmma -c 1 -o $O/prof_lu python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1 > $O/ncu_lu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sk_ -s 3 -c 3 -o $O/prof_sk python tools/sk_probe.py > $O/ncu_sk.log 2>&1
C3C="python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_gemm_dmma -s 4 -c 6 -o $O/prof_gemm $C3C > $O/ncu_gemm.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_schur_inverse -c 2 -o $O/prof_schur $C3C > $O/ncu_schur.log 2>&1
# summaries on the box (the reports themselves exceed what gpurun brings back)
for r in sweep lu sk gemm schur; do
  [ -f $O/prof_$r.ncu-rep ] || continue
  python tools/ncu_summary.py report $O/prof_$r.ncu-rep "round 2 $r" "see tools/prof_round.sh" > $O/summary_$r.txt 2>&1
  for kern in k_sweep_dmma2 k_band_lu_dmma k_sk_parts k_sk_levels k_sk_solve k_gemm_dmma k_schur_inverse; do
    python tools/ncu_inst.py $O/prof_$r.ncu-rep $kern 40 > $O/lines_${r}_$kern.txt 2>/dev/null
    [ -s $O/lines_${r}_$kern.txt ] || rm -f $O/lines_${r}_$kern.txt
  done
  ncu -i $O/prof_$r.ncu-rep --page raw --csv > $O/raw_$r.csv 2>/dev/null
  rm -f $O/prof_$r.ncu-rep
done
ls -la $O
du -sh gpurun_out
