# round-2 evidence run (gpurun): bench lines, launch list and full ncu capture
# of the bench's dominant kernel; summarised into profiles/r02_* afterwards
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/ev3_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/ev3_bench.json 2> gpurun_out/ev3_bench.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/ev3_c1.json 2> gpurun_out/ev3_c1.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-e2e --mode gpu > gpurun_out/ev3_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-e2e --mode gpu > gpurun_out/ev3_ncu_launch.log 2>&1
timeout 300 python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/ev3_p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_omp -c 1 -o gpurun_out/ev3_komp python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/ev3_ncu_full.log 2>&1
echo finished
