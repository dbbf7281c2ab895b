# ncu --set full summaries of the C4 (pivoted) and C2 (narrow solve) kernels on
# the final round-2 build, each only after its command exited 0 without ncu.
set -x
mkdir -p gpurun_out/r02b
O=gpurun_out/r02b
C4="python tools/profile_case.py --n 1000000 --k 64 --nrhs 4 --piv --dd -1.0 --transpose --reps 1"
C2="python tools/profile_case.py --n 1000000 --k 64 --nrhs 1 --dd 1.1 --transpose --reps 1"
timeout 300 $C4 > $O/plain_c4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_band_lu_piv_dmma|k_sweep_piv_dmma|k_sweep_dmma' -c 8 -o $O/prof_c4 $C4 > $O/ncu_c4.log 2>&1
timeout 300 $C2 > $O/plain_c2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_band_lu_dmma|k_sweep_dmma' -c 8 -o $O/prof_c2 $C2 > $O/ncu_c2.log 2>&1
python tools/ncu_summary.py report $O/prof_c4.ncu-rep "Round 2 (final build) - ncu --set full of the C4 pivoted kernels on the BASELINE C4 matrix (no dominance), factorize + solve + transpose solve" "ncu --set full --clock-control none --import-source on -k regex:'k_band_lu_piv_dmma|k_sweep_piv_dmma|k_sweep_dmma' -c 8 $C4" > $O/summary_c4.txt 2>&1
python tools/ncu_summary.py report $O/prof_c2.ncu-rep "Round 2 (final build) - ncu --set full of the C2 kernels (n=1e6, k=64, nrhs=1, dd=1.1), factorize + solve + transpose solve" "ncu --set full --clock-control none --import-source on -k regex:'k_band_lu_dmma|k_sweep_dmma' -c 8 $C2" > $O/summary_c2.txt 2>&1
rm -f $O/*.ncu-rep
timeout 600 python bench.py --config c4 --no-cpu --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c2 --no-cpu --steps 5 > $O/bench_c2.json 2> $O/bench_c2.err
ls -la $O
