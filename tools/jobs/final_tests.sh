timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/fin7_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/fin7_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin7_smoke.log 2>&1; echo "smoke rc=$?"
