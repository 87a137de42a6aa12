mkdir -p gpurun_out
for v in "" rf0; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== variant ${v:-default}" >> gpurun_out/g13.txt
  timeout 120 python tools/variant_bench.py >> gpurun_out/g13.txt 2>&1
  timeout 120 python tools/variant_bench.py >> gpurun_out/g13.txt 2>&1
  timeout 120 python tools/stencil_lag.py 256 >> gpurun_out/g13.txt 2>&1
done
unset SPTRSV_LIB
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -q -x -k "stencil or partition or guard or signed" > gpurun_out/g13_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g13_pytest.log
