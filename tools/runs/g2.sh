python tools/sk_probe.py > gpurun_out/sk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sk_ -s 3 -c 3 -o gpurun_out/prof_sk python tools/sk_probe.py > gpurun_out/ncu_sk.log 2>&1
echo rc=$?
