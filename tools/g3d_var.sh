#!/bin/bash
# 3D stencil variants: per-tile timeline summary + fast/exact kernel medians
o=gpurun_out/t3v; mkdir -p $o; : > $o/res3.txt
for v in "$@"; do
  lib=paper_2012_06959_b200/libsptrsv_b200$v.so
  SPTRSV_LIB=$lib timeout 60 python tools/stencil3d_timeline.py fast > $o/tl.json 2>&1
  tail -1 $o/tl.json | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['lib'].split('/')[-1], 'k', d['kernel_ms'], 'run', d['run_median'], 'zhop', d['zhop_end_median'], 'yhop', d['yhop_end_median'], 'y0z0', round(d['end_Y0_us'][0]-d['ready_Y0_us'][0],1))
" >> $o/res3.txt 2>&1 || tail -3 $o/tl.json >> $o/res3.txt
  SPTRSV_LIB=$lib timeout 60 python tools/variant_bench3d.py >> $o/res3.txt 2>&1
done
