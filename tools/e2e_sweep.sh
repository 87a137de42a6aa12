#!/bin/bash
# e2e of the overlapped host solve vs copy granularity (bands per copy in / out)
for cfg in "1 1" "8 1" "8 4" "8 8" "16 8" "32 16" "4 2"; do
  set -- $cfg
  echo "in=$1 out=$2 $(SPTRSV_STREAM_IN=$1 SPTRSV_STREAM_OUT=$2 timeout 200 python tools/e2e_probe.py 2>&1 | tail -1)"
done
