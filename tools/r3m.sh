for pl in g r m; do
  echo "== plan $pl"; FMP_OMP_PLAN=$pl timeout 600 python bench.py --config 4 --dtype c64 --steps 3 --warmup 2 --no-cpu --no-c3 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('mode'), d.get('mode_step_ms'))"
done
