#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest -x -q --timeout 180 tests/test_replay_gpu.py tests/test_parity_gpu.py tests/test_pdl_gpu.py tests/test_sharded_gpu.py > gpurun_out/r2/pytest_s9.log 2>&1; tail -2 gpurun_out/r2/pytest_s9.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e > gpurun_out/r2/bench9_c4_$i.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r2/bench9_c4_$i.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']['stree_replay_scan']; print('c4', round(d['value']/1e6,2), round(k['us'],3), round(k['frac'],4), 'iso', round(k['isolated_call_us'],2))"; done
