out=gpurun_out/ab.txt; : > $out
for i in 1 2; do
  for d in ab .; do
    (cd $d && timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline) > gpurun_out/bench_ab.log 2>&1
    tail -1 gpurun_out/bench_ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['ms_per_step'])" >> $out 2>&1
  done
done
cat $out
