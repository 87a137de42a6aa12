mkdir -p gpurun_out
cat > /tmp/clk.py <<'PY'
import sys; sys.path.insert(0,'.')
sys.argv=['x']
exec(open('tools/stencil_exp.py').read().split("def main")[0])
for extra in (0, 4, 4|(16<<8), 4|(256<<8)):
    clock(64, extra=extra)
run(64); run(4096)
PY
for v in "" nost xtma; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== variant ${v:-default}" >> gpurun_out/g5.txt
  timeout 300 python /tmp/clk.py >> gpurun_out/g5.txt 2>&1
done
