timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "sparse or support" > gpurun_out/sparse_tests.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/sparse_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --byte-n 0 --no-cpu --tier-n 0 --fp32 0 --single-gate 0 > gpurun_out/sparse_bench.json 2> gpurun_out/sparse_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/sparse_bench.json').read().strip().splitlines()[-1]); a=d['adder']; print(d['value'], a['seconds'], a['first_run_seconds'], a['support_passes'], a['kat_all_ones_R2'])"
