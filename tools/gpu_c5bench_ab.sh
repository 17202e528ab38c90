#!/bin/bash
# C5 bench default vs ${AB_ENV} + GPU tests (run under gpurun)
mkdir -p gpurun_out
timeout 1500 python -m pytest -m gpu -x -q ${AB_TESTS:-tests} > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
for v in "" "$AB_ENV"; do
  tag=$([ -z "$v" ] && echo base || echo ab)
  env $v timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_$tag.log 2>&1
done
echo done
