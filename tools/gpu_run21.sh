cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python bench.py --config c3 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench c3 rc $?
timeout 900 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench c1 rc $?
timeout 600 python -m pytest tests/test_bench_contract.py -q -m gpu 2>&1 | tail -1
