# the driver's bench command, then its ncu launch list, then one full capture of a fused pass (traffic)
bash tools/jobs/bench_full.sh s2c
timeout 3000 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02_launches_bench_s2c.csv python bench.py --steps 20 --warmup 5 > gpurun_out/ncu_launch_s2c.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py gpurun_out/r02_launches_bench_s2c.csv > gpurun_out/r02_launch_summary_s2c.txt 2>&1; head -25 gpurun_out/r02_launch_summary_s2c.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:sv_pass -s 6 -c 1 -o gpurun_out/r02_sv_pass_n32_s2c python bench.py --n 32 --steps 2 --warmup 3 --e2e-steps 0 --adder 0 --byte-n 0 --no-cpu --tier-n 0 --fp32 0 --parity 0 --single-gate 0 > gpurun_out/ncu_full_s2c.log 2>&1; echo "ncu full rc=$?"
