#!/bin/bash
# Round-2 (second pass) measurement: GPU suite, smoke, bench lines for every
# config and the reference arm, the ncu launch list of the default bench
# command, and ncu --set full captures of the headline stencil kernel, the
# band-block solve kernels (TMA sweeps + superblock chain) and the component
# pool on rmat-4M (their DRAM bytes feed profiles/traffic.json).
o=gpurun_out/final5
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "rc=$?" >> $o/smoke.log
timeout 600 python bench.py > $o/bench_default.json 2> $o/bench_default.err
timeout 600 python bench.py --precision exact --no-cpu-baseline > $o/bench_exact.json 2> $o/bench_exact.err
for cfg in lap3d-128 rmat-4M banded-8M lap2d-256; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --steps 100 --warmup 5 --e2e-steps 3 > $o/cfg_$cfg.json 2> $o/cfg_$cfg.err
done
timeout 600 python bench.py --config rmat-4M --precision exact --no-cpu-baseline > $o/cfg_rmat-4M_exact.json 2> $o/cfg_rmat-4M_exact.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_reference.json 2> $o/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_lap2d4096.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $o/ncu_launches.log 2>&1
cap() {  # name regex count run_one-args...
  local name=$1 rx=$2 cnt=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$rx" -c $cnt -o $o/$name -f python tools/run_one.py --reps 1 "$@" > $o/ncu_$name.log 2>&1
  ncu -i $o/$name.ncu-rep --page raw --csv > $o/${name}_raw.csv 2>&1
}
# fast single right-hand side: band groups (no prep tasks), one chain (SPTRSV_ST_GROUP=0: the BD kernel)
cap stencil_fast 'k_stencil2dILb0ELi0ELb0ELi1ELb0ELb0' 1 --config lap2d-4096 --executor stencil --precision fast
ncu -i $o/stencil_fast.ncu-rep --page source --csv --print-source cuda,sass > $o/stencil_fast_source.csv 2>&1
for G in 0 2 4 8; do SPTRSV_ST_GROUP=$G timeout 300 python bench.py --no-cpu-baseline > $o/bench_group$G.json 2> $o/bench_group$G.err; done
cap stencil3d_fast 'k_stencil3d' 1 --config lap3d-128 --executor stencil --precision fast
cap band_fast 'k_bb_sweep_tma|k_bb_chain' 5 --config banded-8M --executor band --precision fast
cap rows_rmat 'k_rowsILi1' 1 --config rmat-4M --executor rows --precision fast
rm -f $o/*.ncu-rep.tmp
exit 0
