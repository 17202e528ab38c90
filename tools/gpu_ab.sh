#!/bin/bash
# A/B iteration: gpu tests, bench (new), bench with $AB_ENV (old), solve launch list
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
env ${AB_ENV} timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_ab.log 2>&1
python tools/prof_step.py --solve-only --steps 1 ${PROF_ARGS} > gpurun_out/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_solve.csv \
    python tools/prof_step.py --solve-only --steps 1 ${PROF_ARGS} > gpurun_out/ncu.log 2>&1
echo done
