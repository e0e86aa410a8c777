mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_facade.py -m gpu -q -x > gpurun_out/r2d_facade.log 2>&1
timeout 300 python tools/c1_latency.py > gpurun_out/r2d_c1lat.log 2>&1
timeout 300 python tools/c1_latency.py pieces >> gpurun_out/r2d_c1lat.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_facade.py::test_facade_reference_recipes -k "not config5_prefix" > gpurun_out/r2d_tests.log 2>&1
echo finished
