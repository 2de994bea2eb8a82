for v in "TPA_SPARSE_DIV=8" "TPA_SPARSE_DIV=8 TPA_NO_POSBITS=1" "TPA_SPARSE_DIV=16" "TPA_SPARSE_DIV=16 TPA_NO_POSBITS=1"; do
  echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
done
