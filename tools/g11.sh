mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "band" > gpurun_out/g11_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g11_pytest.log
timeout 300 python -m pytest tests/test_gpu_baseline_sizes.py -q -x -k "banded" >> gpurun_out/g11_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g11_pytest.log
timeout 300 python bench.py --config banded-8M --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/g11_banded.json 2> gpurun_out/g11_banded.err
