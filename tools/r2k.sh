mkdir -p gpurun_out
b() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-c3 --mode $1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', '$1', round(d['value']), round(d['ms_per_step'],3))"; }
for md in custom:6 custom:8 custom:10 custom:12 custom:14 custom:16; do b $md base; done > gpurun_out/r2k_sweep.log
cp paper_1205_4139_b200/libfmp_cuda.so /tmp/base.so
for v in _variants/*.so; do cp $v paper_1205_4139_b200/libfmp_cuda.so; b custom:10 $v; b custom:14 $v; done >> gpurun_out/r2k_sweep.log
cp /tmp/base.so paper_1205_4139_b200/libfmp_cuda.so
timeout 300 python tools/phases.py 4096 --modes custom:12 > gpurun_out/r2k_phases.log 2>&1
echo finished
