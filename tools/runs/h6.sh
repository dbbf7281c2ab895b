mkdir -p gpurun_out
O=gpurun_out
timeout 600 python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1 > $O/h6_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep_dmma2 -s 2 -c 1 -o $O/h6_sweep python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1 > $O/h6_ncu.log 2>&1
ncu -i $O/h6_sweep.ncu-rep --page source --csv --print-source sass > $O/h6_sweep_sass.csv 2>/dev/null
ncu -i $O/h6_sweep.ncu-rep --page raw --csv > $O/h6_sweep_raw.csv 2>/dev/null
python tools/ncu_inst.py $O/h6_sweep.ncu-rep k_sweep_dmma2 40 > $O/h6_lines.txt 2>&1
ls -la $O | tail
rm -f $O/h6_sweep.ncu-rep
