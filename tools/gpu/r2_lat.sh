#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest -x -q tests/test_replay_gpu.py tests/test_parity_gpu.py tests/test_pdl_gpu.py > gpurun_out/r2/pytest_lat.log 2>&1
tail -5 gpurun_out/r2/pytest_lat.log
for c in c3 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e > gpurun_out/r2/bench_lat_$c.json 2> gpurun_out/r2/bench_lat_$c.err
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-next --no-cpu-baseline --no-e2e --no-fuse > gpurun_out/r2/bench_lat_${c}_nofuse.json 2>> gpurun_out/r2/bench_lat_$c.err
done
