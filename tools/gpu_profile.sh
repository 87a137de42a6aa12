#!/bin/bash
# Round profile pass: bench lines, ncu launch list of the bench command, one
# ncu --set full capture of the stencil kernel (lap2d-4096) and of the chains
# kernel (lap3d-128). Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --precision exact --no-cpu-baseline > gpurun_out/bench_exact.json 2> gpurun_out/bench_exact.err
timeout 600 python bench.py --config lap3d-128 --no-cpu-baseline > gpurun_out/bench_lap3d.json 2> gpurun_out/bench_lap3d.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_lap2d4096.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil2d -c 1 -o gpurun_out/stencil_full -f python tools/run_one.py --config lap2d-4096 --executor stencil --reps 1 > gpurun_out/ncu_full_stencil.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chains -c 1 -o gpurun_out/chains_full -f python tools/run_one.py --config lap3d-128 --executor chains --reps 1 > gpurun_out/ncu_full_chains.log 2>&1
exit 0
