timeout 900 python tools/pass_model.py 33 10 > gpurun_out/pm_cfg10.jsonl 2>&1; tail -1 gpurun_out/pm_cfg10.jsonl
