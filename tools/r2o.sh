mkdir -p gpurun_out
timeout 300 python tools/c1_e2e.py > gpurun_out/r2o_c1e2e.log 2>&1
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/r2o_c1.json 2> gpurun_out/r2o_c1.err
timeout 300 python -m pytest tests -m gpu -q -x -k "latency or abi or facade or small or omp" > gpurun_out/r2o_tests.log 2>&1
echo finished
