T=fin6
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/${T}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
bash tools/jobs/bench_full.sh $T
