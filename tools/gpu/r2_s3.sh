#!/bin/bash
# batch-1 latency anatomy: PDL chain floor + per-CTA timeline of the small-batch kernel
mkdir -p gpurun_out/r2
for n in 80 148 24; do ./tools/pdl_floor $n; done > gpurun_out/r2/pdl_floor.txt 2>&1
cat gpurun_out/r2/pdl_floor.txt
STREE_TRACE=1 python -c "from paper_2505_14969_b200 import build; build.build(force=True)" > /dev/null 2>&1
for f in 7 1; do timeout 120 python tools/trace_lat.py --config c3 --flags $f > gpurun_out/r2/tracelat_c3_f$f.txt 2>&1; done
timeout 120 python tools/trace_lat.py --config c3 --flags 7 --fused 0 > gpurun_out/r2/tracelat_c3_scan.txt 2>&1
timeout 120 python tools/trace_lat.py --config c2 --flags 7 > gpurun_out/r2/tracelat_c2_f7.txt 2>&1
head -3 gpurun_out/r2/tracelat_*.txt
