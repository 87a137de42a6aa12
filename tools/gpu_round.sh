#!/bin/bash
# One GPU-box pass: gpu tests, bench lines, ncu launch list. Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --config lap3d-128 --no-cpu-baseline > gpurun_out/bench_lap3d.json 2> gpurun_out/bench_lap3d.err
timeout 600 python bench.py --precision exact --no-cpu-baseline > gpurun_out/bench_exact.json 2> gpurun_out/bench_exact.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_lap2d4096.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
exit 0
