cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t6_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/t6_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t6_gpu.log 2>&1; echo gpu tests rc $?; tail -3 gpurun_out/t6_gpu.log
for v in "" "TPA_RELABEL=0"; do
  echo "== c2 $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "spmv|ms/batch"
  echo "== c4 $v"; env $v python tools/ab_time.py c4 32 2>&1 | grep -E "spmv|ms/batch"
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench c2 rc $?
timeout 1200 python bench.py --config c5 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench c5 rc $?
TPA_C5=1 timeout 2400 python -m pytest tests/test_c5.py -q -s -x > gpurun_out/t6_c5.log 2>&1; echo c5 rc $?; tail -12 gpurun_out/t6_c5.log
