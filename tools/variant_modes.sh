# bench step time of each build (_variants/*.so and the in-tree one) per mode
# list: VARIANT_MODES="v1.so:gpu,custom:16 base:gpu"
mkdir -p gpurun_out
cp paper_1205_4139_b200/libfmp_cuda.so /tmp/base.so
for spec in $VARIANT_MODES; do
  v=${spec%%:*}; modes=${spec#*:}
  if [ "$v" = base ]; then cp /tmp/base.so paper_1205_4139_b200/libfmp_cuda.so; else cp "_variants/$v" paper_1205_4139_b200/libfmp_cuda.so; fi
  for md in ${modes//,/ }; do
    echo -n "$v $md: "; timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-c3 --mode $md 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3))"
  done
done
cp /tmp/base.so paper_1205_4139_b200/libfmp_cuda.so
