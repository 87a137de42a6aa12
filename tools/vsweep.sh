# lap2d-4096 and lap3d-128 stencil kernel times: default library vs the variants named as arguments
for v in "" "$@"; do
  if [ -n "$v" ]; then export SPTRSV_LIB=$PWD/paper_2012_06959_b200/libsptrsv_b200_$v.so; else unset SPTRSV_LIB; fi
  echo "== variant ${v:-default}"
  timeout 300 python tools/variant_bench.py
  timeout 300 python tools/variant_bench3d.py
done
