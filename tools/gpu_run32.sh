cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for v in default mb16 mb14 default; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== $v"; for c in c2 c4; do env $L python tools/ab_pre.py $c 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"; done
done
