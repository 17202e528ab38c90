#!/bin/bash
# config sweep (run under gpurun): full GPU tests + smoke, then C1-C5 bench lines and the default C2 bench
mkdir -p gpurun_out/sweep
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/sweep/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/sweep/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sweep/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/sweep/smoke.log
for c in C1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sweep/bench_$c.log 2>&1
done
timeout 600 python bench.py --config C2 --layout per_node --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sweep/bench_C2_per_node.log 2>&1
timeout 900 python bench.py > gpurun_out/sweep/bench_C2.log 2>&1
echo done
