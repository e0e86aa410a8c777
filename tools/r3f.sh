mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_wht_fold -c 1 -f -o gpurun_out/r3f_fold_f32 python tools/prof_fold.py f32 > gpurun_out/r3f_f32.log 2>&1
echo finished
