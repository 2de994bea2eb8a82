cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t19_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/t19_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/t19_gpu.log 2>&1; echo gpu tests rc $?; tail -2 gpurun_out/t19_gpu.log; grep FAILED gpurun_out/t19_gpu.log | head
bash tools/profile_round.sh
timeout 1200 python bench.py --config c5 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench c5 rc $?
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo bench ref rc $?
