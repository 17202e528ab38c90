#!/bin/bash
cat gpurun_out/pytest.log
for f in bench bench_ab; do python -c "
import json; d=json.loads(open('gpurun_out/$f.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$f', '%.4g'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'solve %.4f'%r['solve_ms'], 'frac %.3f'%r['frac'])" 2>&1 | tail -1; done
python tools/launches.py gpurun_out/launches_solve.csv 2>&1 | head -${1:-40}
