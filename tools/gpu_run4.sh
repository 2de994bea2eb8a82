cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t4_gpu.log 2>&1; echo gpu tests rc $?; tail -3 gpurun_out/t4_gpu.log
for v in "" "TPA_SPMM=2"; do echo "== B16 $v"; env $v python tools/ab_time.py c2 16 2>&1 | grep -E "sweep |ms/batch"; done
echo "== B32"; python tools/ab_time.py c2 32 2>&1 | grep -E "ms/batch"
TPA_C5=1 timeout 2400 python -m pytest tests/test_c5.py -q -s -x > gpurun_out/t4_c5.log 2>&1; echo c5 rc $?
tail -15 gpurun_out/t4_c5.log
timeout 1200 python bench.py --config c5 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench c5 rc $?
tail -3 gpurun_out/bench_c5.err
