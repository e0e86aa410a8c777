set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/r1_gpu.txt
python bench.py --steps 2 --warmup 1 --no-cpu --no-c3 --mode gpu > gpurun_out/r1_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-c3 --mode gpu > gpurun_out/r1_ncu_launch.log 2>&1
python tools/prof_omp.py --mode custom --batch 296 > gpurun_out/r1_p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_omp -c 1 -o gpurun_out/r1_komp python tools/prof_omp.py --mode custom --batch 296 --reps 1 > gpurun_out/r1_ncu_full.log 2>&1
echo finished
