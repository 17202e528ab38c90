#!/bin/bash
# C5 A/B: launch lists of one stage solve (default vs ${AB_ENV}), parity tests of the many-rhs path (run under gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -x -q tests/test_gpu_scale.py tests/test_gpu_solve.py tests/test_gpu_stepping.py > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
for v in "" "${AB_ENV:-HPSB_NO_GS_PIPE=1}"; do
  tag=$([ -z "$v" ] && echo new || echo old)
  env $v ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/c5_$tag.csv python tools/prof_step.py --config C5 --solve-only --steps 1 --warmup 1 > gpurun_out/ncu_c5_$tag.log 2>&1
  python tools/launches.py gpurun_out/c5_$tag.csv 80 > gpurun_out/c5_$tag.txt 2>&1
done
echo done
