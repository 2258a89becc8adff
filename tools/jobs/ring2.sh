timeout 900 python tools/pass_model.py 33 8 > gpurun_out/pm_cfg8.jsonl 2>&1; tail -1 gpurun_out/pm_cfg8.jsonl
timeout 900 python tools/pass_model.py 33 11 > gpurun_out/pm_cfg11.jsonl 2>&1; tail -1 gpurun_out/pm_cfg11.jsonl
