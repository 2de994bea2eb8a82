#!/bin/bash
# round-2 bench lines: C4 headline (driver args) + reference arm, then C2/C3/C1 lines
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
/usr/bin/time -f "wall %e s" timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "c4 rc $?"; tail -1 gpurun_out/r02_bench_c4.err
/usr/bin/time -f "wall %e s" timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref_c4.json 2> gpurun_out/r02_ref_c4.err; echo "ref rc $?"; tail -1 gpurun_out/r02_ref_c4.err
for c in c2 c3 c1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "$c rc $?"
done
