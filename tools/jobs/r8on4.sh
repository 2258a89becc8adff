SVB200_DEVICES=4 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 8 --qubits-per-gpu 30 --byte-n-multi 30 --steps 3 --warmup 3 > gpurun_out/r8_bench.json 2> gpurun_out/r8_bench.err; echo "bench rc=$?"
tail -c 1200 gpurun_out/r8_bench.json; grep -i "error\|Traceback" gpurun_out/r8_bench.err | head -5
