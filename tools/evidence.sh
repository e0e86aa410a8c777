# Evidence run (gpurun): bench lines, launch list, full ncu captures of the
# bench's dominant kernel and of the config-3 kernels.  Summarise afterwards
# with tools/summarize_profile.py.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/ev_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/ev_c1.json 2> gpurun_out/ev_c1.err
timeout 600 python bench.py --config 4 --dtype c64 --steps 3 --warmup 3 > gpurun_out/ev_c4.json 2> gpurun_out/ev_c4.err
timeout 300 python bench.py --solver cosamp --steps 3 --warmup 3 > gpurun_out/ev_cosamp_c2.json 2> gpurun_out/ev_cosamp_c2.err
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-c3 --mode gpu > gpurun_out/ev_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-c3 --mode gpu > gpurun_out/ev_ncu_launch.log 2>&1
timeout 300 python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/ev_p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_omp -c 1 -o gpurun_out/ev_komp python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/ev_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_update -c 1 -o gpurun_out/ev_fu_f32 python tools/prof_fu.py f32 > gpurun_out/ev_ncu_fu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_update -c 1 -o gpurun_out/ev_fu_f64 python tools/prof_fu.py f64 >> gpurun_out/ev_ncu_fu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wht_fold -c 1 -o gpurun_out/ev_fold_f32 python tools/prof_fold.py f32 > gpurun_out/ev_ncu_fold.log 2>&1
echo finished
