#!/bin/bash
# Round-2 measurement pass: GPU suite, smoke, bench lines for every config and
# the reference arm, the ncu launch list of the default bench command, and one
# ncu --set full capture per executor's solve kernel (raw metrics exported to
# CSV; the 2D stencil's source page for the stall-by-role split).
mkdir -p gpurun_out/final
o=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "rc=$?" >> $o/smoke.log
timeout 600 python bench.py > $o/bench_default.json 2> $o/bench_default.err
timeout 600 python bench.py --precision exact --no-cpu-baseline > $o/bench_exact.json 2> $o/bench_exact.err
for cfg in lap3d-128 rmat-4M banded-8M lap2d-256; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --steps 100 --warmup 5 --e2e-steps 3 > $o/cfg_$cfg.json 2> $o/cfg_$cfg.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_reference.json 2> $o/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_lap2d4096.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $o/ncu_launches.log 2>&1
cap() {  # name regex count run_one-args...
  local name=$1 rx=$2 cnt=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$rx" -c $cnt -o $o/$name -f python tools/run_one.py --reps 1 "$@" > $o/ncu_$name.log 2>&1
  ncu -i $o/$name.ncu-rep --page raw --csv > $o/${name}_raw.csv 2>&1
}
cap stencil_fast 'k_stencil2dILb0ELi0ELb0ELi1ELb0ELb1' 1 --config lap2d-4096 --executor stencil --precision fast
ncu -i $o/stencil_fast.ncu-rep --page source --csv --print-source cuda,sass > $o/stencil_fast_source.csv 2>&1




rm -f $o/*.ncu-rep.tmp
exit 0
