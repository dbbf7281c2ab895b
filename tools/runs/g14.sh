for c in c2 c4 c5; do timeout 900 python bench.py --config $c --no-cpu --steps 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
