nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nvidia-smi topo -m | head -5
free -g; nproc
timeout 300 python tools/hostlink_probe.py 16 > gpurun_out/hostlink.json 2>&1
cat gpurun_out/hostlink.json
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider --durations=20 > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
tail -30 gpurun_out/pytest_gpu2.log
