mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "facade or abi or latency or omp_modes or config1 or small or streamed" > gpurun_out/r2c_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_tests.log
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/r2c_c1.json 2> gpurun_out/r2c_c1.err
echo finished
