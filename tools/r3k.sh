cp paper_1205_4139_b200/libfmp_cuda.so /tmp/base.so
run() { timeout 600 python bench.py --config 4 --dtype c64 --steps 3 --warmup 2 --no-cpu --no-c3 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('mode'), d.get('true_support_recovered'))"; timeout 600 python tools/phases.py 592 --n 16384 --m 4096 --k 128 --iters 256 --dtype c64 --modes adaptive 2>&1 | tail -1; }
for v in _variants/*.so; do
  cp "$v" paper_1205_4139_b200/libfmp_cuda.so
  echo "== $v"; run
  timeout 600 python -m pytest tests/test_gpu_scale_parity.py -m gpu -x -q -k "config4 or c64" 2>&1 | tail -2
done
cp /tmp/base.so paper_1205_4139_b200/libfmp_cuda.so
echo "== in-tree"; run
