cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi topo -m 2>&1 | head -5
python tools/d2h_micro.py 2>&1 | tail -5
python tools/d2h_micro.py local 2>&1 | tail -6
for v in default slim default slim; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== $v"; env $L python tools/ab_time.py c2 32 2>&1 | grep -E "ms/batch"; env $L python tools/ab_time.py c2 16 2>&1 | grep -E "ms/batch"
done
echo "== c3 slim"; TPA_LIB=tools/bin/libtpa_slim.so python tools/ab_time.py c3 64 2>&1 | grep -E "ms/batch"
echo "== c3 default"; python tools/ab_time.py c3 64 2>&1 | grep -E "ms/batch"
TPA_LIB=tools/bin/libtpa_slim.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench c2 rc $?
