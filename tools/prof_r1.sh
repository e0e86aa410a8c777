# Round-1 evidence run (gpurun): bench lines, launch list, one full ncu capture
# of the bench's dominant kernel at the bench batch.  Summarise afterwards with
#   python tools/summarize_profile.py 1 c2 gpurun_out/r1_komp.ncu-rep gpurun_out/r1_launches.csv gpurun_out/r1_bench.json
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/r1_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1_ref.json 2> gpurun_out/r1_ref.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/r1_c1.json 2> gpurun_out/r1_c1.err
timeout 600 python bench.py --config 4 --dtype c64 --steps 3 --warmup 3 > gpurun_out/r1_c4.json 2> gpurun_out/r1_c4.err
timeout 300 python bench.py --solver cosamp --steps 3 --warmup 3 > gpurun_out/r1_cosamp_c2.json 2> gpurun_out/r1_cosamp_c2.err
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-c3 --mode gpu > gpurun_out/r1_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-c3 --mode gpu > gpurun_out/r1_ncu_launch.log 2>&1
timeout 300 python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/r1_p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_omp -c 1 -o gpurun_out/r1_komp python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/r1_ncu_full.log 2>&1
echo finished
