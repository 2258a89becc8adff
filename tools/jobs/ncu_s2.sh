timeout 300 python tools/one_pass.py 32 8 0 8 3
timeout 300 python tools/one_pass.py 32 -1 3 8 3
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k sv_pass -c 1 -o gpurun_out/s2_heavy32 python tools/one_pass.py 32 8 0 8 1 > gpurun_out/ncu_s2_heavy.log 2>&1; tail -2 gpurun_out/ncu_s2_heavy.log
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k sv_pass -c 1 -o gpurun_out/s2_adder32 python tools/one_pass.py 32 -1 3 8 1 > gpurun_out/ncu_s2_adder.log 2>&1; tail -2 gpurun_out/ncu_s2_adder.log
