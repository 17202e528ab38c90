#!/bin/bash
# ncu --set full of kernels matching KREGEX in one solve of CONFIG (run under gpurun)
mkdir -p gpurun_out
ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:${KREGEX}" -c ${KCOUNT:-1} \
  -o gpurun_out/kprof python tools/prof_step.py --config ${CONFIG:-C2} --solve-only --steps 1 --warmup 1 > gpurun_out/ncu_k.log 2>&1
python tools/ncu_summary.py gpurun_out/kprof.ncu-rep > gpurun_out/kprof_full.txt 2>&1
python tools/ncu_lines.py gpurun_out/kprof.ncu-rep "${KLINES:-k_}" 30 > gpurun_out/kprof_lines.txt 2>&1
echo done
