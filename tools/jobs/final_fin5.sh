# final tree: the driver's -m gpu tests and smoke, its 1-GPU bench command, the ncu launch list of
# the same command, one full capture of a fused pass (traffic, source view)
T=fin5
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/${T}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
bash tools/jobs/bench_full.sh $T
timeout 3000 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02_launches_bench_$T.csv python bench.py --steps 20 --warmup 5 > gpurun_out/ncu_launch_$T.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py gpurun_out/r02_launches_bench_$T.csv > gpurun_out/r02_launch_summary_$T.txt 2>&1; head -25 gpurun_out/r02_launch_summary_$T.txt
SVB200_JIT_LINEINFO=1 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:sv_pass -s 6 -c 1 -o gpurun_out/r02_sv_pass_n32_$T python bench.py --n 32 --steps 2 --warmup 3 --e2e-steps 0 --adder 0 --byte-n 0 --no-cpu --tier-n 0 --fp32 0 --parity 0 --single-gate 0 > gpurun_out/ncu_full_$T.log 2>&1; echo "ncu full rc=$?"
