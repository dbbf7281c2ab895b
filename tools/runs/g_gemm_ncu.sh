# ncu --set full of the reduced-system kernels of the C3 step (k_gemm_dmma, k_schur_inverse)
set -x
O=gpurun_out/r02g
mkdir -p $O
C="python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1"
timeout 600 $C > $O/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_gemm_dmma -s 4 -c 6 -o $O/prof_gemm $C > $O/ncu_gemm.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_schur_inverse -c 2 -o $O/prof_schur $C > $O/ncu_schur.log 2>&1
for r in gemm schur; do
  [ -f $O/prof_$r.ncu-rep ] || continue
  python tools/ncu_summary.py report $O/prof_$r.ncu-rep "round 2 $r" "$C" > $O/summary_$r.txt 2>&1
  for kern in k_gemm_dmma k_schur_inverse; do
    python tools/ncu_inst.py $O/prof_$r.ncu-rep $kern 40 > $O/lines_${r}_$kern.txt 2>/dev/null
    [ -s $O/lines_${r}_$kern.txt ] || rm -f $O/lines_${r}_$kern.txt
  done
  ncu -i $O/prof_$r.ncu-rep --page raw --csv > $O/raw_$r.csv 2>/dev/null
  rm -f $O/prof_$r.ncu-rep
done
ls -la $O
