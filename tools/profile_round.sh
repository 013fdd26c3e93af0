#!/bin/bash
# Run under gpurun: ncu evidence for the bench's kernels.
#   1. launch list (per-launch device time, cold-cache/serialised) of the bench command itself
#   2. one --set full capture of the dominant kernel (fused replay+scan) and of the scan / commit kernels
#   3. summaries -> gpurun_out/profile_summary.txt, gpurun_out/traffic.json
set -u
OUT=gpurun_out
mkdir -p $OUT
# launch list of the bench command (our kernels only; the input generation kernels are skipped)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none -k regex:'scan_tc|scan_simt|commit_|build_mask|accept_' -c 400 \
    --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
    > $OUT/ncu_launches.log 2>&1
# the unfused order too (scan-only and commit-only kernels)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none -k regex:'scan_tc|scan_simt|commit_|build_mask|accept_' -c 400 \
    --csv --log-file $OUT/launches_nofuse.csv python bench.py --steps 2 --warmup 1 --no-fuse --no-e2e \
    --no-cpu-baseline > $OUT/ncu_launches_nofuse.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:scan_tc_kernel -s 8 -c 2 \
    -o $OUT/prof_fused python tools/prof_kernels.py --fused > $OUT/ncu_fused.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled \
    -k regex:'scan_tc_kernel.*\)0>' -s 8 -c 1 -o $OUT/prof_scan python tools/prof_kernels.py > $OUT/ncu_scan.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled \
    -k regex:'scan_tc_kernel.*\)2>' -s 8 -c 1 -o $OUT/prof_commit python tools/prof_kernels.py > $OUT/ncu_commit.log 2>&1
python tools/ncu_summary.py $OUT > $OUT/profile_summary.txt 2>&1
cat $OUT/profile_summary.txt
# launch list of bench_next (attention, KV commit, conv, conv commit, MSS) and a --set full
# capture of the tree-attention kernel
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:'attn_|kv_commit|tree_conv|conv_commit|mss_' -c 400 --csv \
    --log-file $OUT/launches_next.csv python tools/prof_attn.py > $OUT/ncu_launches_next.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 4 -c 1 -o $OUT/prof_attn \
    python tools/prof_attn.py > $OUT/ncu_attn.log 2>&1
