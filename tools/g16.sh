mkdir -p gpurun_out
rm -f gpurun_out/g16.txt
timeout 120 python tools/variant_bench.py >> gpurun_out/g16.txt 2>&1
timeout 120 python tools/variant_bench.py >> gpurun_out/g16.txt 2>&1
timeout 120 python tools/stencil_lag.py 256 >> gpurun_out/g16.txt 2>&1
timeout 200 python tools/stencil_exp.py --tasks >> gpurun_out/g16.txt 2>&1
timeout 900 python -m pytest tests/ -m gpu -q -x -k "stencil or partition or guard or signed or smoke or baseline or fuzz" > gpurun_out/g16_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g16_pytest.log
