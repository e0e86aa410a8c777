mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "two_ctas or config2 or omp_modes or headline or golden or multi" > gpurun_out/r2w_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2w_tests.log
timeout 300 python tools/phases.py 4096 --modes custom:12 > gpurun_out/r2w_phases.log 2>&1
FMP_F16_GSMEM=1 timeout 300 python tools/phases.py 4096 --modes custom:12 >> gpurun_out/r2w_phases.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-c3 > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err
FMP_F16_GSMEM=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-c3 > gpurun_out/r2w_bench_g.json 2> gpurun_out/r2w_bench_g.err
echo finished
