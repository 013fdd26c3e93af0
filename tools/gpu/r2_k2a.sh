#!/bin/bash
mkdir -p gpurun_out/r2
timeout 900 python -m pytest -x -q --timeout 300 tests/test_replay_gpu.py tests/test_pdl_gpu.py tests/test_sharded_gpu.py tests/test_opts_gpu.py tests/test_parity_gpu.py 2>&1 | tail -2
timeout 600 python bench.py --no-next --no-cpu-baseline --no-e2e > gpurun_out/r2/bench_k2a.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/r2/bench_k2a.json')); r=d['roofline']
print('value', d['value'], 'frac', r['frac'], 'us', r['kernels']['stree_replay_scan']['us'])"
bash tools/gpu/r2_trk2.sh | grep -E "per layer|start|landed|G ready|acc0|acc1|mma_full0|upd_full0|upd_done0|upd_done1|upd_done3|mma_y0issued0|layer [3-6]"
