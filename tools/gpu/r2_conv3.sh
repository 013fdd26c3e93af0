#!/bin/bash
for cfg in "64 3" "32 3" "24 3" "96 2" "48 2" "160 1" "80 1" "40 1"; do
  set -- $cfg
  echo "ring ${1}KB ctas/SM $2: $(STREE_CONV_RING_KB=$1 STREE_CONV_CTAS_PER_SM=$2 python tools/prof_conv.py 2>&1 | head -1)"
done
