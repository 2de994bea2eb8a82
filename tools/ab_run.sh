for v in "" "TPA_LIB=tools/bin/libtpa_t1k.so" "TPA_LIB=tools/bin/libtpa_t1k6.so" "TPA_LIB=tools/bin/libtpa_t512.so"; do
  echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "spmv"
done
