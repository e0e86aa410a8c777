mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-c3 --mode gpu > gpurun_out/r1_plain.json 2>&1
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/r1_c1.json 2> gpurun_out/r1_c1.err
timeout 300 python bench.py --solver cosamp --config 1 --batch 4096 --steps 3 --warmup 3 > gpurun_out/r1_cosamp_c1.json 2> gpurun_out/r1_cosamp_c1.err
echo finished
