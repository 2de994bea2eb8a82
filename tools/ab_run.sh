python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
for v in "" "TPA_SPARSE_DIV=16" "TPA_SPARSE_DIV=8" "TPA_SPARSE_DIV=4" "TPA_SPARSE_DIV=2"; do
  echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
done
python tools/ab_time.py c3 64 2>&1 | grep -E "sweep |ms/batch"
