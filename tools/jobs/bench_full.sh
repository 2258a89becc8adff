# the driver's 1-GPU bench command; $1 = output tag
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err; echo "rc=$?"
python - "$1" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "frac", d["roofline"]["frac"], "fp64aware", d["roofline"]["fp64_aware"]["frac"], "clocks", d["clocks"])
print("e2e", json.dumps(d["e2e"]))
print("adder", d["adder"]["seconds"], "byte", d["byte_mode"]["sec_per_gate"], "fp32", d["fp32"]["ms_per_step"])
PY
