SVB200_DIRECT_IN=1 SVB200_JIT=1 timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_fp.py -q -x -p no:cacheprovider -k "not torchrun" > gpurun_out/din_tests.log 2>&1; echo "rc=$?" >> gpurun_out/din_tests.log; tail -3 gpurun_out/din_tests.log
SVB200_DIRECT_IN=0 timeout 900 python tools/pass_model.py 33 9 > gpurun_out/pm_din0.jsonl 2>&1; tail -1 gpurun_out/pm_din0.jsonl
SVB200_DIRECT_IN=1 timeout 900 python tools/pass_model.py 33 9 > gpurun_out/pm_din1.jsonl 2>&1; tail -1 gpurun_out/pm_din1.jsonl
