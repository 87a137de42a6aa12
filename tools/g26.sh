mkdir -p gpurun_out; rm -f gpurun_out/g26*
for v in "" s3cp0; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  timeout 120 python tools/variant_bench3d.py >> gpurun_out/g26.txt 2>&1
  timeout 120 python tools/variant_bench3d.py >> gpurun_out/g26.txt 2>&1
done
unset SPTRSV_LIB
timeout 600 python -m pytest tests/ -m gpu -q -x -k "3d or lap3d or stencil or guard or baseline" > gpurun_out/g26_pytest.log 2>&1; echo rc=$? >> gpurun_out/g26_pytest.log
