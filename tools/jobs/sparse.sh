timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "sparse or support" > gpurun_out/sparse_tests.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/sparse_tests.log
