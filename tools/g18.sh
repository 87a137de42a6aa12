mkdir -p gpurun_out; rm -f gpurun_out/g18.txt
for v in "" pp0; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  timeout 120 python tools/variant_bench.py >> gpurun_out/g18.txt 2>&1
  timeout 120 python tools/stencil_timeline.py fast >> gpurun_out/g18.txt 2>&1
  timeout 120 python tools/stencil_timeline.py fast 64 >> gpurun_out/g18.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py tests/test_gpu_baseline_sizes.py -q -x -k "stencil or partition or guard or signed or lap2d" > gpurun_out/g18_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g18_pytest.log
