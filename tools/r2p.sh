mkdir -p gpurun_out
for nt in 128 256; do echo "NT=$nt"; FMP_OMP_NT=$nt timeout 300 python tools/c1_e2e.py 2>&1 | grep "fast\]"; FMP_OMP_NT=$nt timeout 300 python tools/phases.py 1 --kind hadamard --n 1024 --m 256 --k 16 --dtype f64 --modes fast 2>&1; done > gpurun_out/r2p.log
echo finished
