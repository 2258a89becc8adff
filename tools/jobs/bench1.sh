timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "rc=$?"
tail -c 6000 gpurun_out/bench_r02a.json; tail -20 gpurun_out/bench_r02a.err
