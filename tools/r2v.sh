mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "large or apply_adjoint or transform" > gpurun_out/r2v_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2v_tests.log
timeout 300 python tools/prof_large.py --iters 60 > gpurun_out/r2v_p.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2v_launches.csv python tools/prof_large.py --iters 60 > gpurun_out/r2v_ncu.log 2>&1
echo finished
