for b in 0 1; do
SVB200_BULK=$b timeout 300 python tools/one_pass.py 32 0 0 8 3
SVB200_BULK=$b timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k sv_pass -c 1 -o gpurun_out/bulk${b}_p00 python tools/one_pass.py 32 0 0 8 1 > gpurun_out/ncu_bulk$b.log 2>&1; tail -1 gpurun_out/ncu_bulk$b.log
done
