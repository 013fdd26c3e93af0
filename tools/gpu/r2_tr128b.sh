#!/bin/bash
mkdir -p gpurun_out/r2
STREE_TRACE=1 python -c "from paper_2505_14969_b200 import build; build.build(force=True)" > /dev/null 2>&1
timeout 120 python tools/trace_tc128.py --B 16 --T 128 > gpurun_out/r2/trace128_b16.txt 2>&1; head -24 gpurun_out/r2/trace128_b16.txt
grep -E "layer [3-6]" gpurun_out/r2/trace128_b16.txt
timeout 120 python tools/trace_tc128.py --B 16 --T 128 --flags 1 > gpurun_out/r2/trace128_b16_f1.txt 2>&1; head -20 gpurun_out/r2/trace128_b16_f1.txt
