#!/bin/bash
# round-2 evidence pass: full -m gpu suite, smoke, C5 line, C4 ncu (final kernels) + launch list
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $? $(( $(date +%s) - t0 ))s"; tail -2 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r02_smoke.log
t0=$(date +%s); timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err; echo "c5 rc $? $(( $(date +%s) - t0 ))s"
bash tools/profile_c4.sh c4
