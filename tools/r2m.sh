mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "two_ctas or config2 or omp_modes or headline or golden" > gpurun_out/r2m_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2m_tests.log
timeout 300 python tools/phases.py 4096 --modes custom:12 > gpurun_out/r2m_phases.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-c3 --mode custom:12 > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
echo finished
