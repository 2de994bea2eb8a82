cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in c2 c4 c5; do python tools/ab_pre.py $c 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"; done
TPA_MV_TILE_ROWS=256 timeout 900 python -m pytest tests/test_partition.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/t20_gpu.log 2>&1; echo gpu tests rc $?; tail -1 gpurun_out/t20_gpu.log; grep FAILED gpurun_out/t20_gpu.log | head
timeout 900 python bench.py --config c4 --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench c4 rc $?
