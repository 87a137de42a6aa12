#!/bin/bash
# ncu --set full of the two stencil kernels (lap2d-4096 fast, lap3d-128 fast) + source pages for the stall-by-role split
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:k_stencil2dILb0E' -c 1 -o gpurun_out/stencil_full4 -f python tools/run_one.py --config lap2d-4096 --executor stencil --reps 1 > gpurun_out/ncu4_stencil.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:k_stencil3dILb0E' -c 1 -o gpurun_out/stencil3d_full4 -f python tools/run_one.py --config lap3d-128 --executor stencil --reps 1 > gpurun_out/ncu4_stencil3d.log 2>&1
exit 0
