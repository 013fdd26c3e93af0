for v in "16 4" "16 2" "8 4" "8 2" "32 4" "32 2"; do set -- $v
  python -c "from paper_2505_14969_b200 import build as b; b.build(force=True, extra=('-DSTREE_CONV_KC=$1','-DSTREE_CONV_GROUPS=$2'))" > /dev/null 2>&1 || echo build fail $v
  echo "KC=$1 groups=$2"; python tools/prof_conv.py 2>&1 | tail -3
done
python -m paper_2505_14969_b200.build --force > /dev/null 2>&1
