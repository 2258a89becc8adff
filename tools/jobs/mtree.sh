timeout 1200 python -m pytest tests/test_gpu_fp.py tests/test_gpu_ladder.py tests/test_gpu_byte.py -q -x -p no:cacheprovider -k "not torchrun" > gpurun_out/mtree_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/mtree_tests.log
timeout 600 python tools/measure_probe.py 33
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:measure --csv --log-file gpurun_out/mtree_launches.csv python tools/measure_probe.py 33 > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/mtree_launches.csv")) if len(r) > 10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:][-4:]: print(r[ki][:60], r[vi])
PY
timeout 600 python tools/byte_measure_probe.py 32 2>&1 | tail -2
