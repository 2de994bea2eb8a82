#!/bin/bash
# round-2 final pass: full -m gpu suite, C4 headline (driver args) + reference arm, C2 line
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $? $(( $(date +%s) - t0 ))s"; tail -2 gpurun_out/r02_pytest_gpu.log
t0=$(date +%s); timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "c4 rc $? $(( $(date +%s) - t0 ))s"
t0=$(date +%s); timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref_c4.json 2> gpurun_out/r02_ref_c4.err; echo "ref rc $? $(( $(date +%s) - t0 ))s"
timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "c2 rc $?"
