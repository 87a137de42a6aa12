mkdir -p gpurun_out
timeout 120 python tools/variant_bench.py > gpurun_out/g10.txt 2>&1
cat > /tmp/abl.py <<'PY'
import sys; sys.path.insert(0,'.')
sys.argv=['x']
exec(open('tools/stencil_exp.py').read().split("def main")[0])
# probe 32: compute warp alone; ablations (bits 12..15): 1 no staging, 2 no loads, 4 no shuffle, 8 no publish
for extra in (0, 32, 32|(1<<12), 32|(2<<12), 32|(4<<12), 32|(8<<12), 32|(15<<12)):
    clock(64, extra=extra)
PY
timeout 300 python /tmp/abl.py >> gpurun_out/g10.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k 'regex:k_stencil2dILb0ELi0' -c 1 -o gpurun_out/r02_stencil_fast_full -f python tools/run_one.py --config lap2d-4096 --executor stencil --precision fast --reps 1 > gpurun_out/g10_ncu.log 2>&1
