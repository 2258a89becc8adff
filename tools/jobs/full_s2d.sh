timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2d_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/s2d_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2d_smoke.log 2>&1; echo "smoke rc=$?"
bash tools/jobs/bench_full.sh s2d
python -c "
import json; d=json.loads(open('gpurun_out/bench_s2d.json').read().strip().splitlines()[-1]); print(json.dumps(d['adder']['combined_diagonals'])); print(d['adder']['passes'])"
