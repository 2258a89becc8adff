for c in 6 7 8; do timeout 900 python tools/pass_model.py 33 $c > gpurun_out/pm_cfg$c.jsonl 2>&1; tail -1 gpurun_out/pm_cfg$c.jsonl; done
