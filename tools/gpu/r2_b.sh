#!/bin/bash
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e > /tmp/b.json 2>/dev/null; python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']['stree_replay_scan']; print('c4', round(d['value']/1e6,2), round(k['us'],3), round(k['frac'],4))"; done
