#!/bin/bash
# small-batch kernel: one-CTA-per-SM knob vs default (bench c3 / c2), and the straggler table of the fused trace
O=${O:-gpurun_out/lat2}
mkdir -p $O
python -m paper_2505_14969_b200.build > $O/build.log 2>&1 || { echo build failed; exit 1; }
for one in 0 1; do for c in c3 c2; do
  STREE_LAT_ONE_CTA=$one timeout 300 python bench.py --config $c --no-next --no-cpu-baseline --no-e2e > $O/bench_${c}_one$one.json 2> $O/bench_${c}_one$one.err
  timeout 300 python bench.py --config $c --no-fuse --no-next --no-cpu-baseline --no-e2e > $O/bench_${c}_nofuse.json 2> /dev/null
done; done
STREE_TRACE=1 python -m paper_2505_14969_b200.build > /dev/null 2>&1
timeout 120 python tools/trace_lat.py --config c3 --fused 1 --flags 31 --layers 16 > $O/trace_c3_fused.txt 2>&1
STREE_LAT_ONE_CTA=1 timeout 120 python tools/trace_lat.py --config c3 --fused 1 --flags 31 --layers 16 > $O/trace_c3_fused_one.txt 2>&1
python -m paper_2505_14969_b200.build --force > /dev/null 2>&1
for f in $O/bench_*.json; do python -c "
import json;d=json.load(open('$f'));r=d['roofline'];print('$f'.split('/')[-1],round(d['value']/1e6,2),'M nodes/s',{k:round(v.get('us'),3) for k,v in r['kernels'].items()})"; done
