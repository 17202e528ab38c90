#!/bin/bash
# launch list of the bench command's timed region (2 ARK4 steps; ncu serialises, shares not absolutes)
HPSB_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/step_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_step.log 2>&1
python tools/launches.py gpurun_out/step_launches.csv > gpurun_out/step_launches.txt 2>&1
echo done
