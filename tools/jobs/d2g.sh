nvidia-smi --query-gpu=index,name --format=csv
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 tests/dist_gpu_check.py > gpurun_out/d2g_parity.log 2>&1; echo "parity rc=$?"; grep -c "bit-exact=True" gpurun_out/d2g_parity.log; grep "bit-exact=False" gpurun_out/d2g_parity.log | head
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/d2g_bench.json 2> gpurun_out/d2g_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/d2g_bench.json; tail -5 gpurun_out/d2g_bench.err
