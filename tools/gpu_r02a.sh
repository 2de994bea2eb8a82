#!/bin/bash
# round-2 first GPU pass: full -m gpu suite (C4 fixture pending), C4 bench, C4 reference arm
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; free -g >> gpurun_out/lscpu.txt
timeout 1500 python -m pytest tests -m gpu -q -k "not c4" --durations=20 -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc $?"
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err; echo "ref rc $?"
