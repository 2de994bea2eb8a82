for v in "TPA_SPMV=4" "TPA_SPMV=4 TPA_LIB=tools/bin/libtpa_mv46.so" "TPA_SPMV=4 TPA_LIB=tools/bin/libtpa_mv44.so"; do
  echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "spmv"
done
