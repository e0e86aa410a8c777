mkdir -p gpurun_out
timeout 300 python tools/prof_large.py --iters 60 > gpurun_out/r2r_p.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2r_launches.csv python tools/prof_large.py --iters 60 > gpurun_out/r2r_ncu.log 2>&1
echo finished
