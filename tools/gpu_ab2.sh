#!/bin/bash
# A/B: alternate bench runs of the default (A) and with $AB_ENV (B); prints ms/step and solve ms (run under gpurun)
out=gpurun_out/ab.txt; : > $out
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then e=""; else e="${AB_ENV}"; fi
    env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$v.log 2>&1
    tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), 'solve', round(d['roofline']['solve_ms'],4), 'e2e', '%.3e'%d['e2e']['value'])" >> $out 2>&1 || tail -3 gpurun_out/bench_$v.log >> $out
  done
done
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest.log; fi
if [ -n "$TRACE" ]; then
  rm -f gpurun_out/mega.trace
  HPSB_MEGA_TRACE=gpurun_out/mega.trace python tools/prof_step.py --solve-only --steps 1 ${PROF_ARGS} > gpurun_out/trace.log 2>&1
  python tools/mega_trace.py gpurun_out/mega.trace | head -20 > gpurun_out/mega_trace.txt 2>&1
fi
cat $out
