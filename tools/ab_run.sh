python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
TPA_SPMV=1 python -m pytest tests/test_kernel_variants.py -x -q -m gpu -k "SPMV=1" 2>&1 | tail -1
for v in "" "TPA_LIB=tools/bin/libtpa_t4k.so"; do
echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "spmv"
done
