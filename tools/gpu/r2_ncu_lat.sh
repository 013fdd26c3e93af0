#!/bin/bash
mkdir -p gpurun_out/r2
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:lat_kernel -s 20 -c 3 -o gpurun_out/r2/ncu_lat_v4 \
  python bench.py --config c3 --no-fuse --steps 2 --warmup 1 --no-next --no-cpu-baseline --no-e2e --layers 16 > gpurun_out/r2/ncu_lat_v4.log 2>&1
tail -2 gpurun_out/r2/ncu_lat_v4.log
