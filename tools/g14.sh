mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:k_stencil2dILb0ELi0ELb0ELi1' -c 1 -o gpurun_out/r02_stencil_fast_full -f python tools/run_one.py --config lap2d-4096 --executor stencil --precision fast --reps 1 > gpurun_out/g14_ncu.log 2>&1
ncu -i gpurun_out/r02_stencil_fast_full.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_stencil_fast_sass.csv 2>&1
ncu -i gpurun_out/r02_stencil_fast_full.ncu-rep --page raw --csv > gpurun_out/r02_stencil_fast_raw.csv 2>&1
