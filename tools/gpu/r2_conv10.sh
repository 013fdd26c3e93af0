#!/bin/bash
for v in P A1 A2 A3 A; do
  cp varlib/libstree_$v.so paper_2505_14969_b200/libstree.so; touch paper_2505_14969_b200/libstree.so
  echo "$v $(python tools/prof_conv.py 2>&1 | head -1)"
done
