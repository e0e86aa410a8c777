# Round-1 closing evidence (gpurun): bench lines for configs 1-5 and CoSaMP,
# the reference arm, the launch list of the default bench command, full ncu
# captures of k_omp (bench batch), the config-3 kernels, the generator timing.
# Summarise afterwards with tools/summarize_profile.py and tools/summarize_c3.py.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/fe_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/fe_bench.json 2> gpurun_out/fe_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fe_ref.json 2> gpurun_out/fe_ref.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/fe_c1.json 2> gpurun_out/fe_c1.err
timeout 600 python bench.py --config 4 --dtype c64 --steps 3 --warmup 3 > gpurun_out/fe_c4.json 2> gpurun_out/fe_c4.err
timeout 600 python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/fe_c5.json 2> gpurun_out/fe_c5.err
timeout 300 python bench.py --solver cosamp --steps 3 --warmup 3 > gpurun_out/fe_cosamp_c2.json 2> gpurun_out/fe_cosamp_c2.err
timeout 300 python bench.py --solver cosamp --config 1 --steps 3 --warmup 3 > gpurun_out/fe_cosamp_c1.json 2> gpurun_out/fe_cosamp_c1.err
timeout 300 python tools/gen_time.py > gpurun_out/fe_gen_time.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-c3 --mode gpu > gpurun_out/fe_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fe_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-c3 --mode gpu > gpurun_out/fe_ncu_launch.log 2>&1
timeout 300 python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/fe_p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_omp -c 1 -o gpurun_out/fe_komp python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/fe_ncu_full.log 2>&1
for d in f32 f64; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_update -c 1 -o gpurun_out/fe_fu_$d python tools/prof_fu.py $d > gpurun_out/fe_ncu_fu_$d.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wht_fold -c 1 -o gpurun_out/fe_fold_$d python tools/prof_fold.py $d > gpurun_out/fe_ncu_fold_$d.log 2>&1
done
echo finished
