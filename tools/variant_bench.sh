# config-2 bench step time (mode gpu, no CPU / c3 legs) of alternative builds
# of libfmp_cuda.so (_variants/*.so) against the in-tree build
mkdir -p gpurun_out
cp paper_1205_4139_b200/libfmp_cuda.so /tmp/base.so
for v in _variants/*.so; do
  cp "$v" paper_1205_4139_b200/libfmp_cuda.so
  echo "== $v"; timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-c3 --mode ${MODE:-gpu} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
cp /tmp/base.so paper_1205_4139_b200/libfmp_cuda.so
echo "== base"; timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-c3 --mode ${MODE:-gpu} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
