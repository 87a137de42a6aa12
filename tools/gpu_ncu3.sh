#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:k_rowsILi1E' -c 1 -o gpurun_out/rows_rmat_full -f python tools/run_one.py --config rmat-4M --executor rows --reps 1 > gpurun_out/ncu3_rows.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:k_bandILb0E' -c 1 -o gpurun_out/band_full -f python tools/run_one.py --config banded-8M --executor band --reps 1 > gpurun_out/ncu3_band.log 2>&1
exit 0
