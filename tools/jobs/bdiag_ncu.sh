BYTE_PROBE_PROFILE_GATE=40 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/bdiag_launches.csv python tools/byte_probe.py 32 adder > /dev/null 2>&1; echo "rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/bdiag_launches.csv")) if len(r) > 10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]: print(r[ki][:70], r[vi])
PY
BYTE_PROBE_PROFILE_GATE=40 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_byte_diag_apply -c 2 -o gpurun_out/bdiag40 python tools/byte_probe.py 32 adder > gpurun_out/ncu_bdiag.log 2>&1; tail -1 gpurun_out/ncu_bdiag.log
