for lb in 4 3 4 3; do SVB200_LOW_BITS=$lb timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --tier-n 0 --adder 0 --byte-n 0 --parity 0 --single-gate 0 --fp32 0 --cold-e2e 0 --e2e-steps 0 > gpurun_out/lowb_ab.json 2>gpurun_out/lowb_ab.err; python -c "
import json; d=json.loads(open('gpurun_out/lowb_ab.json').read().strip().splitlines()[-1]); print('low $lb', d['ms_per_step'], d['fused_passes_per_step'], d['roofline']['frac'], d['roofline']['fp64_aware']['frac'], d['clocks']['sm_mhz'])"; done
SVB200_LOW_BITS=4 timeout 900 python tools/pass_model.py 33 8 > gpurun_out/pm_low4.jsonl 2>&1; tail -1 gpurun_out/pm_low4.jsonl
SVB200_LOW_BITS=3 timeout 900 python tools/pass_model.py 33 8 > gpurun_out/pm_low3.jsonl 2>&1; tail -1 gpurun_out/pm_low3.jsonl
