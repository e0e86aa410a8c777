mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "not config5_prefix" > gpurun_out/r2x_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2x_tests.log
echo finished
