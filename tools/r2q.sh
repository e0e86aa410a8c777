mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "not config5_prefix" > gpurun_out/r2q_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2q_tests.log
timeout 300 python tools/c1_e2e.py 2>&1 | grep "fast\]" > gpurun_out/r2q_c1.log
timeout 300 python tools/phases.py 1 --kind hadamard --n 1024 --m 256 --k 16 --dtype f64 --modes fast >> gpurun_out/r2q_c1.log 2>&1
timeout 300 python tools/phases.py 4096 --modes custom:12 >> gpurun_out/r2q_c1.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-c3 --mode custom:12 > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
echo finished
