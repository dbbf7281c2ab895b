# end-of-round bench lines on the final build + ncu summaries of the C5 templates
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
# C5's templates (k = 128, nrhs = 32: k_band_lu_dmma<17,17>, k_sweep_dmma<17,*>) on a 2e6-row system
C5C="python tools/profile_case.py --n 2000000 --k 128 --nrhs 32 --reps 1"
timeout 600 $C5C > $O/plain_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep_dmma -c 3 -o $O/prof_c5sweep $C5C > $O/ncu_c5sweep.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_band_lu_dmma -c 1 -o $O/prof_c5lu $C5C > $O/ncu_c5lu.log 2>&1
for r in c5sweep c5lu; do
  [ -f $O/prof_$r.ncu-rep ] || continue
  python tools/ncu_summary.py report $O/prof_$r.ncu-rep "round 2 $r" "$C5C" > $O/summary_$r.txt 2>&1
  for kern in k_sweep_dmma k_band_lu_dmma; do
    python tools/ncu_inst.py $O/prof_$r.ncu-rep $kern 40 > $O/lines_${r}_$kern.txt 2>/dev/null
    [ -s $O/lines_${r}_$kern.txt ] || rm -f $O/lines_${r}_$kern.txt
  done
  rm -f $O/prof_$r.ncu-rep
done
ls -la $O | tail -20
