mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/final2_bench_default.json 2> gpurun_out/final2_bench_default.err
timeout 600 python bench.py --precision exact --no-cpu-baseline > gpurun_out/final2_bench_exact.json 2> /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1
exit 0
