#!/bin/bash
for ms in 32 64 128; do
  for lay in shared per_node; do
    HPSB_MAXSPLIT=$ms timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --layout $lay > gpurun_out/bench_${lay}_$ms.log 2>&1
  done
done
echo done
