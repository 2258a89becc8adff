set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py > gpurun_out/san_$t.log 2>&1; echo "$t rc=$?" >> gpurun_out/san_$t.log
done
tail -3 gpurun_out/*.log
