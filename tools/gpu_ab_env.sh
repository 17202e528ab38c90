#!/bin/bash
# A/B of env settings in this tree: $ENVS is a ';'-separated list of "K=V K=V" settings (run under gpurun)
out=gpurun_out/ab.txt; : > $out
IFS=';' read -ra LIST <<< "${ENVS}"
for i in 1 2; do
  for e in "${LIST[@]}"; do
    env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_ab.log 2>&1
    tail -1 gpurun_out/bench_ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', round(d['ms_per_step'],4), 'solve', round(d['solve']['solve_ms'],4), 'k', ' '.join('%s=%.1f' % (r['kernel'][:12], r['us_per_launch']) for r in d['kernels'][:5]))" >> $out 2>&1 || tail -3 gpurun_out/bench_ab.log >> $out
  done
done
cat $out
