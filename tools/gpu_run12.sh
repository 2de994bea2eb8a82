cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in default mb8 mb7 t1k t1kee mb8ee default; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== $v"; env $L python tools/ab_pre.py c2 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*"; env $L python tools/ab_pre.py c4 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*"
done
