timeout 900 python tools/pass_model.py 32 9 > gpurun_out/pm32.jsonl 2>&1; tail -1 gpurun_out/pm32.jsonl
read L P <<< $(python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/pm32.jsonl") if l.startswith('{"layer')]
r=min(rows, key=lambda r: r["frac"])
print(r["layer"], r["pass"])
PY
)
echo "heaviest: layer $L pass $P"
timeout 300 python tools/one_pass.py 32 $L $P 9 3
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k sv_pass -c 1 -o gpurun_out/heavy32 python tools/one_pass.py 32 $L $P 9 1 > gpurun_out/ncu_heavy.log 2>&1; tail -3 gpurun_out/ncu_heavy.log
