cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in default fxs32 fxs8 default fxs32 fxs8; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== $v"; env $L python tools/ab_pre.py c2 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"; env $L python tools/ab_pre.py c4 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"
done
TPA_LIB=tools/bin/libtpa_fxs32.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_partition.py -q -m gpu -x 2>&1 | tail -1
