mkdir -p gpurun_out/attn
timeout 240 python -m pytest tests/test_attn_gpu.py -x -q > gpurun_out/attn/pytest.log 2>&1; tail -3 gpurun_out/attn/pytest.log
for db in 1 0; do STREE_ATTN_DB=$db timeout 300 python -c "
import sys, json, torch; sys.path.insert(0,'.')
import bench_next
from bench import load_peaks
hbm, bf16, _ = load_peaks()
r = bench_next.measure(torch.device('cuda',0), hbm, bf16)
print('db=$db', json.dumps(r['tree_attn']), 'kv_commit', r['kv_commit']['us'])
"; done
