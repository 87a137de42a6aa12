mkdir -p gpurun_out
cat > /tmp/clk.py <<'PY'
import sys; sys.path.insert(0,'.')
sys.argv=['x']
exec(open('tools/stencil_exp.py').read().split("def main")[0])
for nap in (0, 8, 16, 32, 64):
    clock(64, extra=4 | (nap << 8))
run(64); run(4096); run(4096, "exact")
PY
for v in "" d0s3 d3s5; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== variant ${v:-default}" >> gpurun_out/g6.txt
  timeout 300 python /tmp/clk.py >> gpurun_out/g6.txt 2>&1
done
unset SPTRSV_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py tests/test_gpu_fuzz.py -q -x > gpurun_out/g6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g6_pytest.log
