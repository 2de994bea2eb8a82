python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in "" "TPA_LIB=tools/bin/libtpa_uload.so"; do
  echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
done
