#!/bin/bash
# ncu --set full of the small-batch kernel at c3 (scan-only and fused)
mkdir -p gpurun_out/r2
python -c "from paper_2505_14969_b200 import build; build.build(force=True)" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:lat_kernel -s 20 -c 2 -o gpurun_out/r2/ncu_lat_c3_scan \
  python bench.py --config c3 --no-fuse --steps 2 --warmup 1 --no-next --no-cpu-baseline --no-e2e --layers 16 > gpurun_out/r2/ncu_lat_scan.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lat_kernel -s 20 -c 2 -o gpurun_out/r2/ncu_lat_c3_fused \
  python bench.py --config c3 --steps 2 --warmup 1 --no-next --no-cpu-baseline --no-e2e --layers 16 > gpurun_out/r2/ncu_lat_fused.log 2>&1
tail -3 gpurun_out/r2/ncu_lat_*.log
ls -la gpurun_out/r2/*.ncu-rep
