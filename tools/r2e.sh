mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_facade.py -m gpu -q -x > gpurun_out/r2e_facade.log 2>&1
timeout 300 python tools/c1_e2e.py > gpurun_out/r2e_c1e2e.log 2>&1
echo finished
