#!/bin/bash
# C2 A/B: bench (no CPU leg) default vs ${AB_ENV}, solve launch lists, parity (run under gpurun)
mkdir -p gpurun_out
for v in "" "$AB_ENV"; do
  tag=$([ -z "$v" ] && echo base || echo ab)
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$tag.log 2>&1
  env $v ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python tools/prof_step.py --steps 1 > gpurun_out/ncu_$tag.log 2>&1
  python tools/launches.py gpurun_out/launches_$tag.csv > gpurun_out/launches_$tag.txt 2>&1
done
if [ -n "$AB_TESTS" ]; then env $AB_ENV timeout 900 python -m pytest -m gpu -x -q $AB_TESTS > gpurun_out/pytest_ab.log 2>&1; fi
echo done
