#!/bin/bash
# banded-8M through the N > 1 bench path on one GPU (both ranks time-slice cuda:0)
o=gpurun_out/bp; mkdir -p $o
for N in 2 4; do
SPTRSV_BENCH_SAME_DEVICE=1 SPTRSV_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --config banded-8M --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_n$N.json 2> $o/bench_n$N.err
done
