#!/bin/bash
# C5 (k = 64) launch list of one stage solve with DRAM bytes (run under gpurun)
mkdir -p gpurun_out
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/c5_solve.csv python tools/prof_step.py --config C5 --solve-only --steps 1 --warmup 1 > gpurun_out/ncu_c5.log 2>&1
python tools/launches.py gpurun_out/c5_solve.csv 80 > gpurun_out/c5_solve.txt 2>&1
echo done
