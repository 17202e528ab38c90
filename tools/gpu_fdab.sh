timeout 900 python -m pytest -m gpu -x -q tests/test_gpu_solve.py tests/test_gpu_stepping.py tests/test_gpu_scale.py > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
AB_ENV=HPSB_FD_MMA_FLUX=1 bash tools/gpu_ab_c2.sh
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_new.csv python tools/prof_step.py --config C5 --solve-only --steps 1 --warmup 1 > gpurun_out/ncu_c5.log 2>&1
python tools/launches.py gpurun_out/c5_new.csv 80 > gpurun_out/c5_new.txt 2>&1
