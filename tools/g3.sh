mkdir -p gpurun_out
( time timeout 600 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_records.py -q -x ) > gpurun_out/g3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g3_pytest.log
timeout 300 python bench.py > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
timeout 300 python bench.py --config lap3d-128 --no-cpu-baseline > gpurun_out/g3_bench_lap3d.json 2> gpurun_out/g3_bench_lap3d.err
