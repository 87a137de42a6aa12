#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil2d -c 1 -o gpurun_out/stencil_full2 -f python tools/run_one.py --config lap2d-4096 --executor stencil --reps 1 > gpurun_out/ncu2_stencil.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows -c 1 -o gpurun_out/rows_rmat_full -f python tools/run_one.py --config rmat-4M --executor rows --reps 1 > gpurun_out/ncu2_rows.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_band -c 1 -o gpurun_out/band_full -f python tools/run_one.py --config banded-8M --executor band --reps 1 > gpurun_out/ncu2_band.log 2>&1
exit 0
