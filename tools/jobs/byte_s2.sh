SVB200_TIME_BYTE_PASSES=1 BYTE_PROBE_VERBOSE=1 timeout 600 python tools/byte_probe.py 32 bench > gpurun_out/byte_s2_bench.log 2>&1; tail -45 gpurun_out/byte_s2_bench.log
BYTE_PROBE_VERBOSE=1 timeout 600 python tools/byte_probe.py 32 adder > gpurun_out/byte_s2_adder.log 2>&1; tail -3 gpurun_out/byte_s2_adder.log
