#!/bin/bash
# STREE_TRACE timelines of the small-batch kernel only (c3, flags 31, fused and scan-only)
O=${O:-gpurun_out/lat}
mkdir -p $O
STREE_TRACE=1 python -m paper_2505_14969_b200.build > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 120 python tools/trace_lat.py --config c3 --fused 1 --flags 31 --layers 16 > $O/trace_c3_fused.txt 2>&1
timeout 120 python tools/trace_lat.py --config c3 --fused 0 --flags 31 --layers 16 > $O/trace_c3_scan.txt 2>&1
python -m paper_2505_14969_b200.build --force > /dev/null 2>&1
