#!/bin/bash
timeout 600 python -m pytest -x -q --timeout 180 tests/test_opts_gpu.py tests/test_replay_gpu.py tests/test_sharded_gpu.py 2>&1 | tail -1
for c in c4 c3; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e > /tmp/b.json 2>/dev/null; python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']['stree_replay_scan']; print('$c', round(d['value']/1e6,2), round(k['us'],3), round(k['frac'],4), round(k['isolated_call_us'],2))"; done
