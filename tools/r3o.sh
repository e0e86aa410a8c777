timeout 900 python -m pytest tests/test_gpu_scale_parity.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --no-c3 --no-e2e --mode gpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
timeout 300 python tools/phases.py 1184 --modes custom:8 2>&1 | tail -1
