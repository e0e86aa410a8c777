mkdir -p gpurun_out
timeout 300 python tools/phases.py 1184 --modes custom:8,conventional > gpurun_out/r3a_phases.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_omp -c 1 -f -o gpurun_out/r3a_omp python tools/prof_omp.py --what omp --mode custom --fu 8 --batch 4096 --reps 1 > gpurun_out/r3a_ncu.log 2>&1
echo finished
