for v in 1 0; do
SVB200_LAZY_MEMSET=$v timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 4 --byte-n 0 --no-cpu --tier-n 0 --fp32 0 --single-gate 0 --cold-e2e 0 > gpurun_out/lazy_$v.json 2> gpurun_out/lazy_$v.err; echo "v=$v rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/lazy_$v.json').read().strip().splitlines()[-1]); a=d['adder']; e=d['e2e']; print('v=$v', 'adder', a['seconds'], a['first_run_seconds'], a['support_passes'], 'e2e', e['value'], [c['s'] for c in e['calls']], 'dense', e['dense']['value'])"
done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "support or sparse or adder or golden" > gpurun_out/lazy_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/lazy_tests.log
