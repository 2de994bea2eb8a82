cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t8_gpu.log 2>&1; echo gpu tests rc $?; tail -3 gpurun_out/t8_gpu.log
TPA_RELABEL=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_partition.py -q -m gpu -x > gpurun_out/t8_relabel.log 2>&1; echo relabel tests rc $?; tail -2 gpurun_out/t8_relabel.log
python tools/ab_time.py c2 16 2>&1 | grep -E "sweep |ms/batch"
python tools/ab_time.py c2 32 2>&1 | grep -E "ms/batch"
timeout 1200 python bench.py --config c5 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench c5 rc $?; tail -2 gpurun_out/bench_c5.err
