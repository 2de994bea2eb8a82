cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/t37_gpu.log 2>&1; echo gpu tests rc $?; tail -1 gpurun_out/t37_gpu.log
timeout 900 python bench.py --config c3 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench c3 rc $?
timeout 900 python bench.py --config c4 --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench c4 rc $?
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench c1 rc $?
