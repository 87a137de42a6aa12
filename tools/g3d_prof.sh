#!/bin/bash
# ncu --set full capture of the 3D stencil kernel (fast) with its source page,
# split by warp role.
o=gpurun_out/p3d; mkdir -p $o
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil3d -c 1 -o $o/s3 -f python tools/run_one.py --reps 1 --config lap3d-128 --executor stencil --precision ${1:-fast} > $o/ncu.log 2>&1
ncu -i $o/s3.ncu-rep --page source --csv --print-source cuda,sass > $o/s3_source.csv 2>&1
ncu -i $o/s3.ncu-rep --page raw --csv > $o/s3_raw.csv 2>&1
python tools/ncu_roles.py $o/s3_source.csv paper_2012_06959_b200/csrc/stencil3d.cu > $o/roles.txt 2>&1
rm -f $o/s3.ncu-rep
