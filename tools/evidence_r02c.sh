# Round-2 closing evidence (gpurun): the whole GPU test suite, bench lines for
# configs 1-5 and CoSaMP, the reference arm, the launch list of the default
# bench command, full ncu captures of k_omp (bench batch) and the config-3
# FWHT.  Summarise afterwards with tools/summarize_profile.py.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/ce_gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ce_tests.log 2>&1; tail -2 gpurun_out/ce_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/ce_bench.json 2> gpurun_out/ce_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ce_ref.json 2> gpurun_out/ce_ref.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/ce_c1.json 2> gpurun_out/ce_c1.err
timeout 600 python bench.py --config 4 --dtype c64 --steps 3 --warmup 3 > gpurun_out/ce_c4.json 2> gpurun_out/ce_c4.err
timeout 600 python bench.py --config 4 --dtype c128 --steps 3 --warmup 3 > gpurun_out/ce_c4_c128.json 2> gpurun_out/ce_c4_c128.err
timeout 600 python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/ce_c5.json 2> gpurun_out/ce_c5.err
timeout 300 python bench.py --solver cosamp --steps 3 --warmup 3 > gpurun_out/ce_cosamp_c2.json 2> gpurun_out/ce_cosamp_c2.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-e2e --mode gpu > gpurun_out/ce_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ce_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-c3 --no-e2e --mode gpu > gpurun_out/ce_ncu_launch.log 2>&1
timeout 300 python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/ce_p.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_omp -c 1 -f -o gpurun_out/ce_komp python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/ce_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wht_fold -c 1 -f -o gpurun_out/ce_fold_f32 python tools/prof_fold.py f32 > gpurun_out/ce_ncu_fold_f32.log 2>&1
echo finished
