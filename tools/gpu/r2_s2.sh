#!/bin/bash
# round-2 session-2 baseline: full GPU suite, smoke, bench lines (c4 default, c3, c2)
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu.log 2>&1; tail -3 gpurun_out/r2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; tail -2 gpurun_out/r2/smoke.log
timeout 600 python bench.py > gpurun_out/r2/bench_default.json 2> gpurun_out/r2/bench_default.err; tail -c 600 gpurun_out/r2/bench_default.json
for c in c3 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e --no-fuse > gpurun_out/r2/bench_${c}_nofuse.json 2>> gpurun_out/r2/bench_$c.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/r2/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['roofline'])" 
done
