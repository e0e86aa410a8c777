mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x > gpurun_out/r2u_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2u_tests.log
timeout 300 paper_1205_4139_b200/fmp_driver --config 2 --gpus 1 --steps 5 --warmup 2 > gpurun_out/r2u_driver_c2.json 2>&1
timeout 300 paper_1205_4139_b200/fmp_driver --config 1 --gpus 1 --steps 50 --warmup 5 > gpurun_out/r2u_driver_c1.json 2>&1
echo finished
