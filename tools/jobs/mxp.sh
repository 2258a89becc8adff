timeout 600 python tools/measure_probe.py 33
SVB200_XP_NO_ONES=1 timeout 600 python tools/measure_probe.py 33
SVB200_XP_NO_ONES=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:measure --csv --log-file gpurun_out/mxp_launches.csv python tools/measure_probe.py 33 > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/mxp_launches.csv")) if len(r) > 10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:][-4:]: print(r[ki][:60], r[vi])
PY
