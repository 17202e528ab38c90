#!/bin/bash
# quick GPU iteration with an env A/B (run under gpurun): ENVS=';'-separated settings, tests first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stepping.py tests/test_gpu_solve.py ${IT_TESTS} -m gpu -x -q 2>&1 | tail -4 > gpurun_out/it.txt
IFS=';' read -ra LIST <<< "${ENVS}"
for i in 1 2; do
  for e in "${LIST[@]}"; do
    env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_it.log 2>&1
    tail -1 gpurun_out/bench_it.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', round(d['ms_per_step'],4), 'solve', round(d['solve']['solve_ms'],4), 'parity', d['parity']['ok'], ' '.join('%s=%.1f' % (r['kernel'][:20], r['us_per_launch']) for r in d['kernels'][:8]))" >> gpurun_out/it.txt 2>&1 || tail -5 gpurun_out/bench_it.log >> gpurun_out/it.txt
  done
done
cat gpurun_out/it.txt
