#!/bin/bash
# subtree DMMA kernels: parity tests, then bench A/B against the SIMT kernels, then a solve launch list (run under gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_scale.py tests/test_gpu_hazards.py -m gpu -x -q > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
ENVS="HPSB_NO_SUB_MMA=0;HPSB_NO_SUB_MMA=1" bash tools/gpu_ab_env.sh
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_solve.csv python tools/prof_step.py --solve-only --steps 1 > gpurun_out/ncu.log 2>&1
python tools/launches.py gpurun_out/launches_solve.csv > gpurun_out/launches_solve.txt 2>&1
echo done
