timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2s2_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s2_gputests.log; tail -3 gpurun_out/r2s2_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s2_smoke.log 2>&1; echo "smoke rc=$?"
