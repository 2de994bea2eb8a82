cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for v in default l512 l4k l128; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== $v"; env $L python tools/ab_pre.py c5 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"
done
