mkdir -p gpurun_out; rm -f gpurun_out/g18.txt
for v in "" ard acoef aboth; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  timeout 120 python tools/variant_bench.py >> gpurun_out/g18.txt 2>&1
  timeout 120 python tools/stencil_timeline.py fast >> gpurun_out/g18.txt 2>&1
  timeout 120 python tools/stencil_timeline.py fast 64 >> gpurun_out/g18.txt 2>&1
done

