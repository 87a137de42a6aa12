#!/bin/bash
# Round-2 re-entry check: full GPU suite, smoke, bench lines for every config, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02a_bench_default.json 2> gpurun_out/r02a_bench_default.err
timeout 600 python bench.py --precision exact --no-cpu-baseline > gpurun_out/r02a_bench_exact.json 2> gpurun_out/r02a_bench_exact.err
for cfg in lap3d-128 rmat-4M banded-8M; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/r02a_cfg_$cfg.json 2> gpurun_out/r02a_cfg_$cfg.err
done
exit 0
