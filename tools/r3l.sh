mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3l_tests.log 2>&1; tail -3 gpurun_out/r3l_tests.log
timeout 600 python bench.py --config 4 --dtype c64 --steps 3 --warmup 2 --no-c3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 c64', d['value'], d['ms_per_step'], d.get('mode'), d['cpu_baseline'].get('support_agreement_with_gpu'))"
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-c3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['value'], d['ms_per_step'], d.get('mode'), d['e2e']['value'])"
timeout 300 python bench.py --solver cosamp --steps 3 --warmup 3 --no-c3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cosamp', d['value'], d['ms_per_step'])"
timeout 300 python bench.py --steps 5 --warmup 3 --no-c3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['mode_step_ms'])"
