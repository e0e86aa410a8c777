mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-e2e --mode gpu > gpurun_out/ev3_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-e2e --mode gpu > gpurun_out/ev3_ncu_launch.log 2>&1
echo finished
