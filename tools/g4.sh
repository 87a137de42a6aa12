mkdir -p gpurun_out
for v in "" mb; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== variant ${v:-default}" >> gpurun_out/g4.txt
  timeout 300 python tools/variant_bench.py >> gpurun_out/g4.txt 2>&1
  timeout 300 python tools/stencil_exp.py --tasks >> gpurun_out/g4.txt 2>&1
  timeout 300 python tools/stencil_abl.py 2>&1 | head -1 >> gpurun_out/g4.txt
done
export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_mb.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stencil" > gpurun_out/g4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g4_pytest.log
