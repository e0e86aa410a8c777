cp paper_1205_4139_b200/libfmp_cuda.so /tmp/base.so
for v in _variants/*.so; do
  cp "$v" paper_1205_4139_b200/libfmp_cuda.so
  echo "== $v"; timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --no-c3 --no-e2e --mode gpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
cp /tmp/base.so paper_1205_4139_b200/libfmp_cuda.so
for fu in 4 5 6 7 8 9 10 12 14; do
  echo "== custom:$fu"; timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --no-c3 --no-e2e --mode custom:$fu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
