timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_ladder.py tests/test_gpu_fp.py -q -x -p no:cacheprovider -k "not torchrun" > gpurun_out/perf2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/perf2_tests.log; tail -2 gpurun_out/perf2_tests.log
timeout 900 python tools/pass_model.py 33 9 > gpurun_out/pm_new.jsonl 2>&1; tail -1 gpurun_out/pm_new.jsonl
timeout 1200 python bench.py --steps 20 --warmup 5 --tier-n 0 --no-cpu > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo "rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02b.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step", "fused_passes_per_step")}, d["roofline"]["frac"], d["clocks"], d["fp32"]["ms_per_step"], d["e2e"], d["adder"]["seconds"], d["parity"])
PY
