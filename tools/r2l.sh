mkdir -p gpurun_out
timeout 300 python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/r2l_p.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_omp -c 1 -o gpurun_out/r2l_komp python tools/prof_omp.py --mode gpu --batch 4096 --reps 1 > gpurun_out/r2l_ncu.log 2>&1
echo finished
