mkdir -p gpurun_out; rm -f gpurun_out/g36*
for v in "" ts2 ts6; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== $v" >> gpurun_out/g36.txt
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bb -c 8 --csv python tools/run_one.py --config banded-8M --executor band --precision fast --reps 2 2>/dev/null | grep -E "k_bb|kernel_ms" | cut -c1-40,150-400 >> gpurun_out/g36.txt
  timeout 600 python tools/run_one.py --config banded-8M --executor band --precision fast --reps 3 2>&1 | grep kernel_ms >> gpurun_out/g36.txt
done
