mkdir -p gpurun_out
timeout 120 python tools/variant_bench.py >> gpurun_out/g9.txt 2>&1
timeout 120 python tools/stencil_exp.py --tasks 2>&1 >> gpurun_out/g9.txt
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py tests/test_gpu_fuzz.py -q -x -k "stencil or partition or fuzz or guard or signed" > gpurun_out/g9_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g9_pytest.log
