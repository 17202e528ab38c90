#!/bin/bash
# round-2 closing evidence (run under gpurun): GPU tests + smoke, bench lines of every config, the reference arm,
# C2 launch list with DRAM bytes, ncu --set full of the step's kernels with k_mega's source lines, C5 solve launch list
O=gpurun_out/final3
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_C2.log 2>&1
HPSB_LAYOUT=per_node timeout 900 python bench.py --no-cpu-baseline > $O/bench_C2_per_node.log 2>&1
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1
done
timeout 900 python bench.py --plain-fields --no-cpu-baseline > $O/bench_C2_plain_fields.log 2>&1
timeout 1700 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_C2_reference.log 2>&1
HPSB_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/c2_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
python tools/launches.py $O/c2_bench_launches.csv > $O/c2_bench_launches.txt 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k "regex:k_mega|k_leaf_fd_mma|k_sub_up|k_sub_down" -c 8 \
  -o $O/c2_step_kernels python tools/prof_step.py --steps 1 > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/c2_step_kernels.ncu-rep > $O/c2_step_kernels_full.txt 2>&1
python tools/ncu_lines.py $O/c2_step_kernels.ncu-rep k_mega 25 > $O/c2_k_mega_source_lines.txt 2>&1
rm -f $O/c2_step_kernels.ncu-rep
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/c5_solve.csv python tools/prof_step.py --config C5 --solve-only --steps 1 --warmup 1 > $O/ncu_c5.log 2>&1
python tools/launches.py $O/c5_solve.csv 80 > $O/c5_solve_launches.txt 2>&1
rm -f gpurun_out/mega.trace
HPSB_MEGA_TRACE=gpurun_out/mega.trace timeout 300 python tools/prof_step.py --solve-only --steps 1 --warmup 0 > $O/trace.log 2>&1
python tools/mega_trace.py gpurun_out/mega.trace > $O/mega_trace.txt 2>&1
echo done
