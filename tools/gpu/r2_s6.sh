#!/bin/bash
# full GPU suite + c4/c3/c2 bench lines + c3 trace
mkdir -p gpurun_out/r2
timeout 900 python -m pytest -x -q --timeout 120 tests -m gpu > gpurun_out/r2/pytest_s6.log 2>&1
tail -3 gpurun_out/r2/pytest_s6.log
for c in c4 c3 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e > gpurun_out/r2/bench6_$c.json 2> gpurun_out/r2/bench6_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/r2/bench6_$c.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print('$c', round(d['value']/1e6,2), 'M nodes/s', {n: round(v['us'],3) for n, v in k.items()}, 'frac', round(d['roofline']['frac'],3))"
done
bash tools/gpu/r2_tr.sh
