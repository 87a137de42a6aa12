mkdir -p gpurun_out; rm -f gpurun_out/g41*
for prec in exact fast; do
  timeout 600 python tools/run_one.py --config rmat-4M --executor rows --precision $prec --reps 4 2>&1 | grep kernel_ms | tail -2 >> gpurun_out/g41.txt
done
timeout 900 python -m pytest tests/ -m gpu -q -x -k "rows or rmat or fuzz or parity or records or partition or multiproc or baseline or debug" > gpurun_out/g41_pytest.log 2>&1; echo rc=$? >> gpurun_out/g41_pytest.log
