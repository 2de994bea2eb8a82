python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
for v in "" "TPA_LIB=tools/bin/libtpa_mb9.so"; do
echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
env $v python tools/ab_time.py c3 64 2>&1 | grep -E "ms/batch"
done
