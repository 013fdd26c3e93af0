#!/bin/bash
mkdir -p gpurun_out/r2; python -c "from paper_2505_14969_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 600 python tools/sweep_c5.py > gpurun_out/r2/sweep_c5_v3.txt 2>&1; grep -E "T64|T128|T256" gpurun_out/r2/sweep_c5_v3.txt | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['case'], round(d['packed_us'],2), d.get('packed_b16_nodes_per_s'))"
