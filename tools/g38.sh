mkdir -p gpurun_out; rm -f gpurun_out/g38*
for v in "" bbd pf24; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== $v" >> gpurun_out/g38.txt
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_bb -c 4 --csv python tools/run_one.py --config banded-8M --executor band --precision fast --reps 1 2>/dev/null | grep -E "k_bb" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-30,60-200 >> gpurun_out/g38.txt
  timeout 600 python tools/run_one.py --config banded-8M --executor band --precision fast --reps 3 2>&1 | grep kernel_ms >> gpurun_out/g38.txt
done
unset SPTRSV_LIB
timeout 600 python -m pytest tests/ -m gpu -q -x -k "band" > gpurun_out/g38_pytest.log 2>&1; echo rc=$? >> gpurun_out/g38_pytest.log
