timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/sup2_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/sup2_gputests.log
timeout 900 python tools/adder_combine_probe.py 16
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu --tier-n 0 --byte-n 0 --parity 0 --single-gate 0 --fp32 0 > gpurun_out/sup2_bench.json 2>gpurun_out/sup2_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/sup2_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step']); print(json.dumps(d['e2e'])[:900]); a=d['adder']; print(a['seconds'], a.get('dense_seconds'), a.get('support'), a['combined_diagonals']['seconds'])"
