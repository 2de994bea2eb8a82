cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for i in 1 2; do
  python tools/ab_pre.py c2 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"; python tools/ab_pre.py c4 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"
done
python tools/ab_pre.py c5 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_partition.py tests/test_kernel_variants.py -q -m gpu -x 2>&1 | tail -2
