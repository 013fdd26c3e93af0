#!/bin/bash
# tree conv: register cap (min CTAs per SM) so that two layers' CTAs can be resident under PDL
for mb in 10 13 16; do
  python -c "from paper_2505_14969_b200 import build as b; b.build(force=True, extra=('-DSTREE_CONV_MINB=$mb',))" > /dev/null 2>&1 || echo build fail $mb
  echo "minb=$mb"; python tools/prof_conv.py 2>&1 | tail -1
done
timeout 300 python -m pytest tests/test_conv_gpu.py -q -x 2>&1 | tail -1
python -m paper_2505_14969_b200.build --force > /dev/null 2>&1
