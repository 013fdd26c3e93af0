#!/bin/bash
mkdir -p gpurun_out/r2
STREE_TRACE=1 python -c "from paper_2505_14969_b200 import build; build.build(force=True)" > /dev/null 2>&1
STREE_LAT_ONE_CTA=1 timeout 120 python tools/trace_lat.py --config c3 --flags 15 --fused 0 > gpurun_out/r2/tracelat5_c3_scan_1cta_dry.txt 2>&1
timeout 120 python tools/trace_lat.py --config c3 --flags 15 --fused 0 > gpurun_out/r2/tracelat5_c3_scan_dry.txt 2>&1
tail -25 gpurun_out/r2/tracelat5_c3_scan_1cta_dry.txt; head -1 gpurun_out/r2/tracelat5_c3_scan_dry.txt
