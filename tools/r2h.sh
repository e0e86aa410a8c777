# evidence: sanitizers over every kernel family, config 4 c128 / c64 (full-batch
# agreement with the reference library), config 5, CoSaMP config 2
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_small.py quick > gpurun_out/r2h_san_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/r2h_san_$tool.log
done
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 > gpurun_out/r2h_c5.json 2> gpurun_out/r2h_c5.err
timeout 900 python bench.py --config 4 --dtype c128 --steps 3 --warmup 3 > gpurun_out/r2h_c4_c128.json 2> gpurun_out/r2h_c4_c128.err
timeout 1200 python bench.py --config 4 --dtype c64 --steps 3 --warmup 3 --cpu-sample 2048 > gpurun_out/r2h_c4_c64_full.json 2> gpurun_out/r2h_c4_c64_full.err
echo finished
