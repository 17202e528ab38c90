#!/bin/bash
# A/B/C...: bench in each source tree listed in $DIRS (built in place), interleaved, 3 rounds (run under gpurun)
out=gpurun_out/ab.txt; : > $out
for i in 1 2 3; do
  for d in ${DIRS}; do
    (cd $d && env ${AB_ENV} timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS}) > gpurun_out/bench_ab.log 2>&1
    tail -1 gpurun_out/bench_ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', round(d['ms_per_step'],4), 'solve', round(d['solve']['solve_ms'],4), 'mega', round(d['roofline']['us_per_launch'],1), 'e2e', '%.3e'%d['e2e']['value'])" >> $out 2>&1 || tail -3 gpurun_out/bench_ab.log >> $out
  done
done
sort $out
