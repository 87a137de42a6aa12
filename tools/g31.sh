mkdir -p gpurun_out; rm -f gpurun_out/g31*
for v in "" 1; do
  if [ -n "$v" ]; then export SPTRSV_NO_BD=1; else unset SPTRSV_NO_BD; fi
  echo "== NO_BD=$v" >> gpurun_out/g31.txt
  timeout 120 python tools/variant_bench.py >> gpurun_out/g31.txt 2>&1
  timeout 120 python tools/variant_bench.py >> gpurun_out/g31.txt 2>&1
  timeout 120 python tools/stencil_timeline.py fast >> gpurun_out/g31.txt 2>&1
done
unset SPTRSV_NO_BD
timeout 900 python -m pytest tests/ -m gpu -q -x -k "stencil or lap2d or partition or guard or signed or baseline or fuzz or many or e2e or stream or smoke or debug" > gpurun_out/g31_pytest.log 2>&1; echo rc=$? >> gpurun_out/g31_pytest.log
