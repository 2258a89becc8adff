SVB200_DIRECT_OUT=1 SVB200_DIRECT_IN=2 SVB200_JIT=1 timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_ladder.py -q -x -p no:cacheprovider > gpurun_out/direct_tests.log 2>&1; echo "rc=$?" >> gpurun_out/direct_tests.log; tail -2 gpurun_out/direct_tests.log
SVB200_DIRECT_OUT=1 timeout 900 python tools/pass_model.py 33 9 > gpurun_out/pm_do1.jsonl 2>&1; tail -1 gpurun_out/pm_do1.jsonl
SVB200_DIRECT_OUT=1 SVB200_DIRECT_IN=1 timeout 900 python tools/pass_model.py 33 9 > gpurun_out/pm_do1_di1.jsonl 2>&1; tail -1 gpurun_out/pm_do1_di1.jsonl
SVB200_DIRECT_OUT=1 SVB200_DIRECT_IN=2 timeout 900 python tools/pass_model.py 33 9 > gpurun_out/pm_do1_di2.jsonl 2>&1; tail -1 gpurun_out/pm_do1_di2.jsonl
