mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_omp -c 1 -f -o gpurun_out/r3j_omp python tools/prof_omp.py --what omp --mode custom --fu 8 --batch 4096 --reps 1 > gpurun_out/r3j_ncu.log 2>&1
echo finished
