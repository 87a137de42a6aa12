#!/bin/bash
# ncu --set full of the exact-mode 2D stencil kernel (speculative Markstein), lap2d-4096
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:k_stencil2dILb1E' -c 1 -o gpurun_out/stencil_exact_full5 -f python tools/run_one.py --config lap2d-4096 --executor stencil --precision exact --reps 1 > gpurun_out/ncu5_stencil_exact.log 2>&1
exit 0
