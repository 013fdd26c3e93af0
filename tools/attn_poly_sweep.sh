#!/bin/bash
# K7b: share of the softmax exponentials computed by the FMA-pipe polynomial (STREE_ATTN_DB_POLY = n: every n-th pair)
for n in 0 4 3 2; do
  python -c "from paper_2505_14969_b200 import build as b; b.build(force=True, extra=('-DSTREE_ATTN_DB_POLY=$n',))" > /dev/null 2>&1 || echo build fail $n
  timeout 300 python -m pytest tests/test_attn_gpu.py -q -x -k "hyb8b or ragged or chain" 2>&1 | tail -1
  timeout 300 python -c "
import sys, json, torch; sys.path.insert(0,'.')
import bench_next
from bench import load_peaks
hbm, bf16, _ = load_peaks()
r = bench_next.measure(torch.device('cuda',0), hbm, bf16)
print('poly=$n', round(r['tree_attn']['us'], 2), round(r['tree_attn']['frac'], 3))
"
done
python -m paper_2505_14969_b200.build --force > /dev/null 2>&1
