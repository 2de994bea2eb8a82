cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t29_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/t29_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/t29_gpu.log 2>&1; echo gpu tests rc $?; tail -1 gpurun_out/t29_gpu.log; grep FAILED gpurun_out/t29_gpu.log | head
for c in c2 c4 c5; do python tools/ab_pre.py $c 2>&1 | tail -1 | grep -o "spmv.*ms [0-9.]*\|Error.*"; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench c2 rc $?
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print(d['value'], d['ms_per_step'], d['roofline']['spmv']['avg_ms'], d['e2e']['value'], d['clocks'])"
