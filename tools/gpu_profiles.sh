#!/bin/bash
# round profiles: config sweep, bench-command launch list, ncu --set full of one solve per layout
mkdir -p gpurun_out/prof
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_$c.log 2>&1
done
timeout 300 python bench.py --config C2 --layout per_node --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_C2_per_node.log 2>&1
timeout 600 python bench.py > gpurun_out/prof/bench_C2.log 2>&1
# launch list of the bench command itself (timed region only)
HPSB_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/prof/c2_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_bench.log 2>&1
python tools/launches.py gpurun_out/prof/c2_bench_launches.csv > gpurun_out/prof/c2_bench_launches.txt 2>&1
for lay in shared per_node; do
  ncu --profile-from-start off --set full --clock-control none --import-source on \
    -o gpurun_out/prof/c2_solve_$lay python tools/prof_step.py --solve-only --steps 1 --layout $lay > gpurun_out/prof/ncu_full_$lay.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof/c2_solve_$lay.ncu-rep > gpurun_out/prof/c2_solve_ncu_full_$lay.txt 2>&1
done
echo done
