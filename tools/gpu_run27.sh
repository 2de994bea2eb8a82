cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in default th128 default th128; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== $v"; for c in c2 c4; do env $L python tools/ab_pre.py $c 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"; done
done
echo "== c5 th128"; TPA_LIB=tools/bin/libtpa_th128.so python tools/ab_pre.py c5 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"
TPA_LIB=tools/bin/libtpa_th128.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py -q -m gpu -x 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_partition.py -q -m gpu -x 2>&1 | tail -1
