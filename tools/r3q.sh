mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:k_omp -c 1 -f -o /tmp/r3q_c4 python tools/prof_c4.py 592 > gpurun_out/r3q_ncu.log 2>&1
ncu -i /tmp/r3q_c4.ncu-rep --page raw --csv > gpurun_out/r3q_c4_raw.csv 2>/dev/null
ls -la gpurun_out/
