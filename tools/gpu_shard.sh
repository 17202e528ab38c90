#!/bin/bash
# sharding iteration: new tests first, then the whole gpu suite, bench, and the
# multi-rank bench code path on one GPU (gloo; numbers not reportable)
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_shard.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
HPSB_BENCH_DEVICE=0 HPSB_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config C1 \
  --steps 3 --warmup 3 > gpurun_out/bench_gloo2.log 2>&1
echo done
