for m in 2 3; do SVB200_XP_MINB8=$m timeout 900 python tools/pass_model.py 33 8 > gpurun_out/pm_minb$m.jsonl 2>&1; tail -1 gpurun_out/pm_minb$m.jsonl; done
