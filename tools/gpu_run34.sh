cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in "" "TPA_BENCH_PROFILE_TIMED=1" "" "TPA_BENCH_PROFILE_TIMED=1"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['value'],1), round(d['ms_per_step'],3), round(r['avg_launch_ms'],4), round(r['share_of_step'],3), round(r['spmv']['avg_ms'],4), d['gpu_launches'])"
done
timeout 600 python -m pytest tests/test_bench_contract.py -q -m gpu 2>&1 | tail -1
