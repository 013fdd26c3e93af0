#!/bin/bash
# Run under gpurun: ncu evidence for the bench's kernels (round 2).
#   1. launch lists (per-launch device time + DRAM bytes, cold-cache/serialised) of the bench commands:
#      c4 fused (the headline), c4 unfused, c3 and c2 (the small-batch kernel), the §8(f) rows
#   2. --set full captures of the dominant kernels (c4 fused, c3 fused small-batch, tree attention)
#   3. summaries -> $OUT/profile_summary.txt, $OUT/traffic.json
set -u
OUT=${OUT:-gpurun_out/prof}
mkdir -p $OUT
REGEX='scan_tc|scan_simt|lat_kernel|commit_|build_mask|accept_'
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --cache-control none -k regex:"$REGEX" -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-next > $OUT/ncu_launches.log 2>&1
ncu --metrics $M --clock-control none --cache-control none -k regex:"$REGEX" -c 400 --csv --log-file $OUT/launches_nofuse.csv \
    python bench.py --steps 2 --warmup 1 --no-fuse --no-e2e --no-cpu-baseline --no-next > $OUT/ncu_launches_nofuse.log 2>&1
for cfg in c3 c2; do
  ncu --metrics $M --clock-control none --cache-control none -k regex:"$REGEX" -c 400 --csv --log-file $OUT/launches_$cfg.csv \
      python bench.py --config $cfg --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-next > $OUT/ncu_launches_$cfg.log 2>&1
done
ncu --set full --clock-control none --cache-control none --import-source on -k regex:scan_tc_kernel -s 8 -c 2 \
    -o $OUT/prof_fused python tools/prof_kernels.py --fused > $OUT/ncu_fused.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lat_kernel -s 20 -c 2 -o $OUT/prof_lat_c3 \
    python bench.py --config c3 --steps 2 --warmup 1 --no-next --no-cpu-baseline --no-e2e --layers 16 > $OUT/ncu_lat.log 2>&1
ncu --metrics $M,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:'attn_|kv_commit|tree_conv|conv_commit|mss_' -c 400 --csv \
    --log-file $OUT/launches_next.csv python tools/prof_attn.py > $OUT/ncu_launches_next.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 4 -c 1 -o $OUT/prof_attn \
    python tools/prof_attn.py > $OUT/ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tree_conv -s 8 -c 1 -o $OUT/prof_conv \
    python tools/prof_conv.py --ncu > $OUT/ncu_conv.log 2>&1
python tools/ncu_summary.py $OUT > $OUT/profile_summary.txt 2>&1
tail -40 $OUT/profile_summary.txt
