timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err; echo "bench rc=$?"
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 20 --warmup 5 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:sv_pass -s 6 -c 1 -o gpurun_out/r02_sv_pass_n32 python bench.py --n 32 --steps 2 --warmup 3 --e2e-steps 0 --adder 0 --byte-n 0 --no-cpu --tier-n 0 --fp32 0 --parity 0 --single-gate 0 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -c 3000 gpurun_out/bench_r02c.json
