cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bench_contract.py -q -m gpu 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'])"
python tools/profile_step.py --config c5 --batch 16 --batches 1 > gpurun_out/c5p_plain.log 2>&1; echo c5 plain rc $?
timeout 1500 ncu --replay-mode application --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:"k_mm_fused" -s 1 -c 2 --csv --log-file gpurun_out/c5_last_traffic.csv python tools/profile_step.py --config c5 --batch 16 --batches 1 > gpurun_out/c5_ncu3.log 2>&1; echo ncu c5 rc $?
tail -12 gpurun_out/c5_last_traffic.csv
