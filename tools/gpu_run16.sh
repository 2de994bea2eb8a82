cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t16_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/t16_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/t16_gpu.log 2>&1; echo gpu tests rc $?; tail -3 gpurun_out/t16_gpu.log; grep FAILED gpurun_out/t16_gpu.log | head
bash tools/profile_round.sh > gpurun_out/t16_profile.log 2>&1; echo profile rc $?; head -5 gpurun_out/t16_profile.log
