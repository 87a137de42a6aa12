mkdir -p gpurun_out
for v in "" cp0; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== variant ${v:-default}" >> gpurun_out/g7.txt
  timeout 300 python tools/nap_sweep.py fast 0 16 32 64 128 >> gpurun_out/g7.txt 2>&1
  timeout 300 python tools/nap_sweep.py exact 16 64 >> gpurun_out/g7.txt 2>&1
  timeout 300 python tools/stencil_exp.py --tasks 2>&1 | head -3 >> gpurun_out/g7.txt
done
unset SPTRSV_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -q -x > gpurun_out/g7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g7_pytest.log
