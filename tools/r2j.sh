mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "two_ctas or config2 or omp_modes or headline or golden or smoke" > gpurun_out/r2j_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2j_tests.log
timeout 300 python tools/phases.py 4096 --modes custom:16,conventional > gpurun_out/r2j_phases.log 2>&1
FMP_OMP_F16=0 timeout 300 python tools/phases.py 4096 --modes custom:16 >> gpurun_out/r2j_phases.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-c3 > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
echo finished
