timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
