SVB200_LOW_BITS=3 SVB200_JIT=1 timeout 900 python -m pytest tests/test_gpu_jit.py -q -x -p no:cacheprovider > gpurun_out/lb_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lb_tests.log; tail -2 gpurun_out/lb_tests.log
for b in 5 4 3; do SVB200_LOW_BITS=$b timeout 900 python tools/pass_model.py 33 9 > gpurun_out/pm_lb$b.jsonl 2>&1; tail -1 gpurun_out/pm_lb$b.jsonl; done
