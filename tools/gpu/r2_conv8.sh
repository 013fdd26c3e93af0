#!/bin/bash
for v in kc8 kc16 kc32; do
  cp varlib/libstree_$v.so paper_2505_14969_b200/libstree.so; touch paper_2505_14969_b200/libstree.so
  echo "$v $(python tools/prof_conv.py 2>&1 | head -1)"
done
timeout 600 python -m pytest -x -q --timeout 300 tests/test_conv_gpu.py 2>&1 | tail -1
