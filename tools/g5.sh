mkdir -p gpurun_out
for md in fast custom:16 custom:24 custom:32 conventional; do echo -n "$md: "; timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-c3 --mode $md 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), d['config']['fast_until'])"; done > gpurun_out/g5_modes.log
timeout 600 python -m pytest tests -m gpu -x -q -k "two_ctas or config2 or omp_modes" > gpurun_out/g5_tests.log 2>&1
