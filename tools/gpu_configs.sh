#!/bin/bash
# Bench lines for every BASELINE config on one GPU (parity configs included).
mkdir -p gpurun_out
for cfg in lap2d-256 lap3d-128 rmat-4M banded-8M; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/cfg_$cfg.json 2> gpurun_out/cfg_$cfg.err
done
exit 0
