mkdir -p gpurun_out; rm -f gpurun_out/g19*
timeout 900 python -m pytest tests/ -m gpu -q -x -k "rows or fuzz or rmat or record or parity or partition or multiproc or baseline" > gpurun_out/g19_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g19_pytest.log
timeout 600 python bench.py --config rmat-4M --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps 2 > gpurun_out/g19_rmat.json 2> gpurun_out/g19_rmat.err
timeout 600 python bench.py --config rmat-4M --precision exact --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/g19_rmat_exact.json 2> gpurun_out/g19_rmat_exact.err
timeout 600 python tools/rows_levels.py > gpurun_out/g19_levels.txt 2>&1
