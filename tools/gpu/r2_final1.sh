#!/bin/bash
# round-2 evidence pass 1: full GPU suite, smoke, default bench line, c2/c3 bench lines, ncu profiles
mkdir -p gpurun_out/r2e
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2e/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2e/pytest_gpu.log 2>&1; tail -2 gpurun_out/r2e/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e/smoke.log 2>&1; tail -1 gpurun_out/r2e/smoke.log
timeout 900 python bench.py > gpurun_out/r2e/bench_default.json 2> gpurun_out/r2e/bench_default.err; tail -c 400 gpurun_out/r2e/bench_default.json
for c in c3 c2; do timeout 600 python bench.py --config $c --no-next > gpurun_out/r2e/bench_$c.json 2> gpurun_out/r2e/bench_$c.err; done
timeout 600 python bench.py --force-heads --no-next --no-cpu-baseline > gpurun_out/r2e/bench_forceheads.json 2> gpurun_out/r2e/bench_forceheads.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2e/bench_reference.json 2> gpurun_out/r2e/bench_reference.err
OUT=gpurun_out/r2e/prof timeout 2400 bash tools/profile_round.sh > gpurun_out/r2e/profile.log 2>&1; tail -30 gpurun_out/r2e/profile.log
