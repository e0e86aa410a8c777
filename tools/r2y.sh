mkdir -p gpurun_out
b() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-c3 --mode $1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['ms_per_step'],3))"; }
for md in custom:1 custom:4 custom:6 custom:8 custom:10 custom:12 custom:16; do b $md; done > gpurun_out/r2y_sweep.log
echo finished
