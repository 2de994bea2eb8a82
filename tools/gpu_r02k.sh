#!/bin/bash
# round-2 final evidence pass (same commands as the driver's round-end tiers)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $? $(( $(date +%s) - t0 ))s"; tail -2 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r02_smoke.log
t0=$(date +%s); timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "c4 rc $? $(( $(date +%s) - t0 ))s"
t0=$(date +%s); timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref_c4.json 2> gpurun_out/r02_ref_c4.err; echo "ref rc $? $(( $(date +%s) - t0 ))s"
