#!/bin/bash
cat gpurun_out/pytest.log
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('value %.4g  ms/step %.3f  solve_ms %.4f  frac %.3f  e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['solve_ms'], d['roofline']['frac'], d['e2e']['value']))"
python tools/launches.py gpurun_out/launches_solve.csv ${1:-0}
