mkdir -p gpurun_out; rm -f gpurun_out/g40*
for v in "" g2 g8 g16; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  for prec in fast exact; do
    echo "== $v $prec" >> gpurun_out/g40.txt
    timeout 600 python tools/run_one.py --config rmat-4M --executor rows --precision $prec --reps 4 2>&1 | grep kernel_ms | tail -2 >> gpurun_out/g40.txt
  done
done
