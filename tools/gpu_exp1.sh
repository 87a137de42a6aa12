#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 300 python tools/stencil_exp.py > gpurun_out/stencil_run.log 2>&1
timeout 300 python tools/stencil_exp.py --tasks > gpurun_out/stencil_tasks.log 2>&1
timeout 300 python tools/stencil_exp.py --clock > gpurun_out/stencil_clock.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil2d -c 1 -o gpurun_out/stencil_full python tools/run_one.py --config lap2d-4096 --executor stencil --reps 1 > gpurun_out/ncu_full_stencil.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chains -c 1 -o gpurun_out/chains_full python tools/run_one.py --config lap3d-128 --executor chains --reps 1 > gpurun_out/ncu_full_chains.log 2>&1
exit 0
