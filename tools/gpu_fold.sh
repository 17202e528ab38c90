#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -3 > gpurun_out/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
HPSB_NO_FOLD=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nofold.log 2>&1
timeout 300 python tools/host_probe.py C2 > gpurun_out/host_probe.log 2>&1
python tools/prof_step.py --solve-only --steps 1 > gpurun_out/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_solve.csv \
    python tools/prof_step.py --solve-only --steps 1 > gpurun_out/ncu.log 2>&1
echo done
