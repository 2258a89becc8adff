timeout 600 python tools/e2e_probe.py 33 > gpurun_out/e2e1_probe.log 2>&1; tail -4 gpurun_out/e2e1_probe.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --tier-n 0 --adder 0 --byte-n 0 --parity 0 --single-gate 0 --cold-e2e 1 > gpurun_out/e2e1_bench.json 2> gpurun_out/e2e1_bench.err; echo "rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/e2e1_bench.json').read().strip().splitlines()[-1]); print(json.dumps(d['e2e'])); print(d['ms_per_step'])"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --tier-n 0 --adder 0 --byte-n 0 --parity 0 --single-gate 0 --fp32 0 --cold-e2e 0 --e2e-steps 4 > gpurun_out/e2e1_bench2.json 2> gpurun_out/e2e1_bench2.err; echo "rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/e2e1_bench2.json').read().strip().splitlines()[-1]); print(json.dumps(d['e2e']))"
