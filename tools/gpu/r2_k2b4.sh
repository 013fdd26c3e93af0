#!/bin/bash
mkdir -p gpurun_out/r2k
timeout 900 python -m pytest -x -q --timeout 300 tests/test_scan_tc128_gpu.py tests/test_opts_gpu.py tests/test_pdl_gpu.py 2>&1 | tail -2
bash tools/gpu/r2_tr128b.sh 2>&1 | grep -E "graph of|landed|jumping|modes|prologue done|G ready|head [0-7] ready|end:|layer [45]"
python -c "from paper_2505_14969_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 600 python tools/sweep_c5.py > gpurun_out/r2k/sweep_c5.txt 2>&1; grep -E "T128|T256|T64" gpurun_out/r2k/sweep_c5.txt | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['case'], round(d['packed_us'],2), d.get('packed_b16_nodes_per_s'))"
