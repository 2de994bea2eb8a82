#!/bin/bash
# A/B of cache-hint variants (tools/bin/libtpa_*.so) on the C2 / C3 query batch.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for v in default gh1 gh2 gh3 st1 gh1st1 gh3st1 default; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== $v"; env $L python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
done
for v in default gh1 gh3 st1; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== c3 $v"; env $L python tools/ab_time.py c3 64 2>&1 | grep -E "ms/batch"
done
