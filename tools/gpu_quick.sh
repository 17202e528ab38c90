#!/bin/bash
# quick GPU iteration: C2 bench (no CPU leg), solve launch list, optional mega trace (run under gpurun)
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_solve.csv python tools/prof_step.py --solve-only --steps 1 ${PROF_ARGS} > gpurun_out/ncu.log 2>&1
python tools/launches.py gpurun_out/launches_solve.csv > gpurun_out/launches_solve.txt 2>&1
if [ -n "$TRACE" ]; then
  rm -f gpurun_out/mega.trace
  HPSB_MEGA_TRACE=gpurun_out/mega.trace python tools/prof_step.py --solve-only --steps 1 > gpurun_out/trace.log 2>&1
  python tools/mega_trace.py gpurun_out/mega.trace > gpurun_out/mega_trace.txt 2>&1
fi
echo done
