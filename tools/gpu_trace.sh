rm -f gpurun_out/mega.trace
HPSB_MEGA_TRACE=gpurun_out/mega.trace python tools/prof_step.py --solve-only --steps 1 > gpurun_out/trace.log 2>&1
python tools/mega_trace.py gpurun_out/mega.trace > gpurun_out/mega_trace.txt 2>&1
