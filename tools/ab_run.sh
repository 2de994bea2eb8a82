python -m pytest tests/test_gpu_parity.py tests/test_topk.py -x -q -m gpu 2>&1 | tail -1
for v in "" "TPA_NO_SEED_PUSH=1"; do
echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
env $v python tools/ab_time.py c3 64 2>&1 | grep -E "ms/batch"
done
