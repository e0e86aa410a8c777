mkdir -p gpurun_out
timeout 300 python tools/phases.py 4096 --modes custom:16,fast,conventional > gpurun_out/r2b_phases.log 2>&1
FMP_OMP_CTAS=1 timeout 300 python tools/phases.py 4096 --modes custom:16 >> gpurun_out/r2b_phases.log 2>&1
echo finished
