cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in default r256 default r256; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== $v"; env $L python tools/ab_pre.py c2 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"; env $L python tools/ab_pre.py c4 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"
done
echo "== c5 r256"; TPA_LIB=tools/bin/libtpa_r256.so python tools/ab_pre.py c5 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"
TPA_LIB=tools/bin/libtpa_r256.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_partition.py -q -m gpu -x 2>&1 | tail -1
