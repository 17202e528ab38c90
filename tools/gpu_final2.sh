#!/bin/bash
# round-2 final evidence (run under gpurun): GPU tests + smoke, C2 bench, C2 launch list with DRAM bytes,
# ncu --set full of the step's main kernels, C5 launch list
mkdir -p gpurun_out/final2
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/final2/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/final2/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final2/smoke.log
timeout 900 python bench.py > gpurun_out/final2/bench_C2.log 2>&1
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final2/bench_C5.log 2>&1
HPSB_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/final2/c2_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final2/ncu_bench.log 2>&1
python tools/launches.py gpurun_out/final2/c2_bench_launches.csv > gpurun_out/final2/c2_bench_launches.txt 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k "regex:k_mega|k_leaf_fd_mma|k_sub_up|k_sub_down|k_root_dir" -c 8 \
  -o gpurun_out/final2/c2_step_kernels python tools/prof_step.py --steps 1 > gpurun_out/final2/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/final2/c2_step_kernels.ncu-rep > gpurun_out/final2/c2_step_kernels_full.txt 2>&1
python tools/ncu_lines.py gpurun_out/final2/c2_step_kernels.ncu-rep k_mega 25 > gpurun_out/final2/c2_k_mega_source_lines.txt 2>&1
rm -f gpurun_out/final2/c2_step_kernels.ncu-rep
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/final2/c5_solve.csv python tools/prof_step.py --config C5 --solve-only --steps 1 --warmup 1 > gpurun_out/final2/ncu_c5.log 2>&1
python tools/launches.py gpurun_out/final2/c5_solve.csv 80 > gpurun_out/final2/c5_solve_launches.txt 2>&1
ncu --profile-from-start off --set full --clock-control none -k "regex:k_deep" -c 2 \
  -o gpurun_out/final2/c5_deep python tools/prof_step.py --config C5 --solve-only --steps 1 --warmup 1 > gpurun_out/final2/ncu_c5_full.log 2>&1
python tools/ncu_summary.py gpurun_out/final2/c5_deep.ncu-rep > gpurun_out/final2/c5_deep_full.txt 2>&1
rm -f gpurun_out/final2/c5_deep.ncu-rep
echo done
