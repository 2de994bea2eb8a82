cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t9_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/t9_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t9_gpu.log 2>&1; echo gpu tests rc $?; tail -3 gpurun_out/t9_gpu.log
timeout 1200 python bench.py --config c5 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench c5 rc $?; tail -2 gpurun_out/bench_c5.err
TPA_C5=1 timeout 2400 python -m pytest tests/test_c5.py -q -s -x > gpurun_out/t9_c5.log 2>&1; echo c5 rc $?; tail -12 gpurun_out/t9_c5.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench c2 rc $?
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/ll_plain.json 2> gpurun_out/ll_plain.err && \
  TPA_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ll_ncu.log 2>&1; echo "launch list rc $?"
python tools/profile_step.py > gpurun_out/ps_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_step_spmv2" -s 30 -c 1 \
      -o gpurun_out/prof_spmv python tools/profile_step.py > gpurun_out/ps_ncu1.log 2>&1; echo "spmv full rc $?"
python tools/profile_step.py --batch 16 > gpurun_out/ps16_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_mm_fused" -s 2 -c 2 \
      -o gpurun_out/prof_b16 python tools/profile_step.py --batch 16 --batches 1 > gpurun_out/ps_ncu2.log 2>&1; echo "b16 full rc $?"
