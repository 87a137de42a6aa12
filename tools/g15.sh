mkdir -p gpurun_out
for v in "" cl2 cl4 cl8; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== variant ${v:-default}" >> gpurun_out/g15.txt
  timeout 120 python tools/variant_bench.py >> gpurun_out/g15.txt 2>&1
  timeout 120 python tools/stencil_lag.py 256 >> gpurun_out/g15.txt 2>&1
done
