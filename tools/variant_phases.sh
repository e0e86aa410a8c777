# phase breakdown of alternative builds of libfmp_cuda.so (_variants/*.so)
for v in _variants/*.so; do
  cp paper_1205_4139_b200/libfmp_cuda.so /tmp/base.so
  cp "$v" paper_1205_4139_b200/libfmp_cuda.so
  echo "== $v"; timeout 300 python tools/phases.py 1184 2>&1 | tail -1
  cp /tmp/base.so paper_1205_4139_b200/libfmp_cuda.so
done
echo "== base"; timeout 300 python tools/phases.py 1184 2>&1 | tail -1
