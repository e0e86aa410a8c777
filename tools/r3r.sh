cp paper_1205_4139_b200/libfmp_cuda.so /tmp/base.so
run() { timeout 600 python bench.py --config 4 --dtype c64 --steps 4 --warmup 2 --no-cpu --no-c3 --no-e2e --mode adaptive 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; }
for v in _variants/*.so; do
  cp "$v" paper_1205_4139_b200/libfmp_cuda.so
  echo "== $v"; run
done
cp /tmp/base.so paper_1205_4139_b200/libfmp_cuda.so
echo "== in-tree (8x4)"; run
