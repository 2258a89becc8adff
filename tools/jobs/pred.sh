timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "support or sparse or golden or ladder or adder or oracle or jit or engine" > gpurun_out/pred_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pred_tests.log
for v in 1 0; do
SVB200_LAZY_PRED=$v timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 4 --byte-n 0 --no-cpu --tier-n 0 --fp32 0 --single-gate 0 --cold-e2e 0 > gpurun_out/pred_$v.json 2> gpurun_out/pred_$v.err; echo "v=$v rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/pred_$v.json').read().strip().splitlines()[-1]); a=d['adder']; e=d['e2e']; print('v=$v', 'adder', a['seconds'], a['first_run_seconds'], 'e2e', e['value'], [c['s'] for c in e['calls']], 'dense', e['dense']['value'], 'parity', d.get('parity',{}).get('oracle_bit_exact', d.get('parity')))" 2>&1 | cut -c1-600
done
