mkdir -p gpurun_out; rm -f gpurun_out/g32*
for v in "" nobd; do
  if [ -n "$v" ]; then export SPTRSV_NO_BD=1; else unset SPTRSV_NO_BD; fi
  echo "== $v" >> gpurun_out/g32.txt
  timeout 120 python tools/variant_bench.py >> gpurun_out/g32.txt 2>&1
  timeout 120 python tools/stencil_timeline.py fast >> gpurun_out/g32.txt 2>&1
done
