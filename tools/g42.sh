mkdir -p gpurun_out; rm -f gpurun_out/g42*
for v in "" ex0; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== $v" >> gpurun_out/g42.txt
  timeout 120 python tools/variant_bench.py >> gpurun_out/g42.txt 2>&1
  timeout 120 python tools/variant_bench.py >> gpurun_out/g42.txt 2>&1
done
unset SPTRSV_LIB
timeout 900 python -m pytest tests/ -m gpu -q -x -k "stencil or lap2d or guard or signed or baseline or fuzz or parity" > gpurun_out/g42_pytest.log 2>&1; echo rc=$? >> gpurun_out/g42_pytest.log
