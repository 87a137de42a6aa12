#!/bin/bash
# End-of-round measurement pass: GPU tests, smoke, bench lines (all configs), ncu launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final_bench_default.json 2> gpurun_out/final_bench_default.err
timeout 600 python bench.py --precision exact --no-cpu-baseline > gpurun_out/final_bench_exact.json 2> /dev/null
for cfg in lap3d-128 rmat-4M banded-8M lap2d-256; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/final_cfg_$cfg.json 2> /dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_lap2d4096.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_reference.json 2> gpurun_out/final_bench_reference.err
exit 0
