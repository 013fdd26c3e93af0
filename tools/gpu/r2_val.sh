#!/bin/bash
mkdir -p gpurun_out/r2v
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/r2v/pytest_gpu.log 2>&1; tail -2 gpurun_out/r2v/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2v/bench_default.json 2> gpurun_out/r2v/bench_default.err; python -c "
import json; d=json.load(open('gpurun_out/r2v/bench_default.json')); r=d['roofline']; n=d['next_rows']
print('value', d['value'], 'frac', r['frac'], 'us', r['kernels']['stree_replay_scan']['us'])
print('k2b', n['c5_sweep'].get('k2b_B16_T128'))
for k in ('tree_attn','tree_conv'): print(k, n[k]['us'], n[k]['frac'])
"
