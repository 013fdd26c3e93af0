#!/bin/bash
mkdir -p gpurun_out/r2
STREE_TRACE=1 python -c "from paper_2505_14969_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 120 python tools/trace_lat.py --config c3 --flags 31 --fused 0 > gpurun_out/r2/tracelat3_c3_scan.txt 2>&1
timeout 120 python tools/trace_lat.py --config c3 --flags 31 > gpurun_out/r2/tracelat3_c3_f15.txt 2>&1
cat gpurun_out/r2/tracelat3_c3_scan.txt | tail -28
