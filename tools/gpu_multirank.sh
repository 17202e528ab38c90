#!/bin/bash
# the multi-rank bench path on one GPU (gloo, both ranks on cuda:0; not for reported numbers)
mkdir -p gpurun_out
for c in C2 C5; do
  HPSB_BENCH_BACKEND=gloo HPSB_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29531 bench.py --config $c --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/multirank_$c.log 2>&1
  echo "rc=$?" >> gpurun_out/multirank_$c.log
done
echo done
