mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "two_ctas or config2 or omp_modes or headline or golden or latency" > gpurun_out/r2t_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2t_tests.log
timeout 300 python tools/phases.py 4096 --modes custom:12 > gpurun_out/r2t_phases.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-c3 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2t_c1.json 2> gpurun_out/r2t_c1.err
echo finished
