timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
python tools/c3_streams.py > gpurun_out/c3s.log 2>&1
python tools/profile_case.py --n 1000000 --k 160 --nrhs 160 --transpose --reps 3 --prof > gpurun_out/prof_c3.log 2>&1
