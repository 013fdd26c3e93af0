#!/bin/bash
# round-2 baseline: batch-1 configs (c2, c3) bench lines + c3 per-CTA trace
set -x
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
for c in c3 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e --no-fuse > gpurun_out/r2/bench_${c}_nofuse.json 2>> gpurun_out/r2/bench_$c.err
done
STREE_TRACE=1 python -c "from paper_2505_14969_b200 import build; build.build()"
for f in 0 7; do
  timeout 120 python tools/trace_tc.py --config c3 --flags $f > gpurun_out/r2/trace_c3_f$f.txt 2>&1
done
timeout 120 python tools/trace_tc.py --config c2 --flags 7 > gpurun_out/r2/trace_c2_f7.txt 2>&1
