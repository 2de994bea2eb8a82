cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t7_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/t7_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t7_gpu.log 2>&1; echo gpu tests rc $?; tail -3 gpurun_out/t7_gpu.log
for v in 0 1; do TPA_RELABEL=$v python tools/ab_pre.py c2 2>&1 | tail -1; done
for v in 0 1; do TPA_RELABEL=$v python tools/ab_pre.py c4 2>&1 | tail -1; done
for v in 0 1; do TPA_RELABEL=$v python tools/ab_pre.py c5 2>&1 | tail -1; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench c2 rc $?
timeout 1200 python bench.py --config c5 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench c5 rc $?; tail -2 gpurun_out/bench_c5.err
