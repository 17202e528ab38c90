#!/bin/bash
# bench (C2) + reference arm + launch list with dram bytes + ncu --set full of k_mega in the step (run under gpurun)
mkdir -p gpurun_out/prof
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/prof/bench_C2.log 2>&1
echo "bench rc=$?" >> gpurun_out/prof/bench_C2.log
if [ -n "$REF" ]; then
  timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/prof/ref_C2.log 2>&1
  echo "ref rc=$?" >> gpurun_out/prof/ref_C2.log
fi
HPSB_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/prof/c2_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_bench.log 2>&1
python tools/launches.py gpurun_out/prof/c2_bench_launches.csv > gpurun_out/prof/c2_bench_launches.txt 2>&1
if [ -n "$FULL" ]; then
  ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_mega -c 2 \
    -o gpurun_out/prof/c2_step_k_mega python tools/prof_step.py --steps 1 > gpurun_out/prof/ncu_full.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof/c2_step_k_mega.ncu-rep > gpurun_out/prof/c2_step_k_mega_full.txt 2>&1
fi
echo done
