mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_wht_fold -c 1 -f -o gpurun_out/r3e_fold_f32 python tools/prof_fold.py f32 > gpurun_out/r3e_f32.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_wht_fold -c 1 -f -o gpurun_out/r3e_fold_f64 python tools/prof_fold.py f64 > gpurun_out/r3e_f64.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fast_update -c 1 -f -o gpurun_out/r3e_fu_f32 python tools/prof_omp.py --what c3fast --dtype f32 --batch 1024 --reps 1 > gpurun_out/r3e_fu.log 2>&1
echo finished
