mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r3i_tests.log 2>&1; tail -3 gpurun_out/r3i_tests.log
for wr in 64 48 40 32 16 0; do
  echo "== wrows $wr"; FMP_F16_WROWS=$wr timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-c3 --no-e2e --mode gpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
timeout 300 python tools/phases.py 1184 --modes custom:8 2>&1 | tail -1
