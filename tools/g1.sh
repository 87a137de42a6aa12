mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/g1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g1_pytest.log
timeout 300 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
