#!/bin/bash
# round-2 results: config sweep, C2 bench (default command) + reference arm, launch list with dram bytes,
# ncu --set full of the step's main kernels (run under gpurun)
mkdir -p gpurun_out/final
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_$c.log 2>&1
done
timeout 600 python bench.py --config C2 --layout per_node --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_C2_per_node.log 2>&1
timeout 900 python bench.py > gpurun_out/final/bench_C2.log 2>&1
HPSB_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/final/c2_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final/ncu_bench.log 2>&1
python tools/launches.py gpurun_out/final/c2_bench_launches.csv > gpurun_out/final/c2_bench_launches.txt 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k "regex:k_mega|k_leaf_fd_mma|k_sub_up|k_sub_down|k_root_dir" -c 8 \
  -o gpurun_out/final/c2_step_kernels python tools/prof_step.py --steps 1 > gpurun_out/final/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/final/c2_step_kernels.ncu-rep > gpurun_out/final/c2_step_kernels_full.txt 2>&1
python tools/ncu_lines.py gpurun_out/final/c2_step_kernels.ncu-rep k_mega 25 > gpurun_out/final/c2_k_mega_source_lines.txt 2>&1
rm -f gpurun_out/final/c2_step_kernels.ncu-rep
echo done
