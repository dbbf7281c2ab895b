python tools/sk_check.py 64 1 1 4 1.5 > gpurun_out/skc.log 2>&1
python tools/sk_check.py 64 1 1 2 1.5 >> gpurun_out/skc.log 2>&1
python tools/sk_check.py 200 2 2 4 1.5 >> gpurun_out/skc.log 2>&1
python tools/sk_probe.py 1024 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sk_ -s 3 -c 3 -o gpurun_out/prof_sk2 python tools/sk_probe.py 1024 > gpurun_out/ncu_sk.log 2>&1
