mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not config5_prefix" > gpurun_out/r2s_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2s_tests.log
timeout 300 python tools/phases.py 4096 --modes custom:12 > gpurun_out/r2s_phases.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-c3 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
echo finished
