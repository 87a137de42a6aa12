mkdir -p gpurun_out
for v in "" cl2 cl4 cl8; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== variant ${v:-default}" >> gpurun_out/g12.txt
  timeout 120 python tools/variant_bench.py >> gpurun_out/g12.txt 2>&1
  timeout 120 python tools/stencil_lag.py 256 >> gpurun_out/g12.txt 2>&1
done
unset SPTRSV_LIB
cat > /tmp/abl.py <<'PY'
import sys; sys.path.insert(0,'.')
sys.argv=['x']
exec(open('tools/stencil_exp.py').read().split("def main")[0])
for extra in (0, 32, 32|(1<<12), 32|(2<<12), 32|(4<<12), 32|(8<<12), 32|(3<<12), 32|(15<<12)):
    clock(64, extra=extra)
PY
echo "== ablations" >> gpurun_out/g12.txt
timeout 300 python /tmp/abl.py >> gpurun_out/g12.txt 2>&1
