#!/bin/bash
timeout 600 python -m pytest -x -q --timeout 180 tests/test_scan_tc128_gpu.py tests/test_opts_gpu.py 2>&1 | tail -1
bash tools/gpu/r2_tr128.sh 2>&1 | grep -E "graph of|prologue|head 0 built|head 1 built|head 2 built|acc head 2|head 2 done|end:" 
timeout 600 python tools/sweep_c5.py > gpurun_out/r2/sweep_c5_v3.txt 2>&1; grep -E "T128|T256" gpurun_out/r2/sweep_c5_v3.txt | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['case'], round(d['packed_us'],2), d.get('packed_b16_nodes_per_s'))"
