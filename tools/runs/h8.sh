mkdir -p gpurun_out
O=gpurun_out
timeout 600 python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1 > $O/h8_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep_dmma2 -s 2 -c 1 -o $O/h8_sweep python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 1 > $O/h8_ncu.log 2>&1
ncu -i $O/h8_sweep.ncu-rep --page source --csv --print-source sass > $O/h8_sweep_sass.csv 2>/dev/null
ncu -i $O/h8_sweep.ncu-rep --page raw --csv > $O/h8_sweep_raw.csv 2>/dev/null
rm -f $O/h8_sweep.ncu-rep
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_band_lu_dmma -c 1 -o $O/h8_lu python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --factor-only --reps 1 > $O/h8_ncu_lu.log 2>&1
ncu -i $O/h8_lu.ncu-rep --page source --csv --print-source sass > $O/h8_lu_sass.csv 2>/dev/null
ncu -i $O/h8_lu.ncu-rep --page raw --csv > $O/h8_lu_raw.csv 2>/dev/null
python tools/ncu_inst.py $O/h8_lu.ncu-rep k_band_lu_dmma 60 > $O/h8_lu_lines.txt 2>&1
rm -f $O/h8_lu.ncu-rep
ls -la $O | tail
