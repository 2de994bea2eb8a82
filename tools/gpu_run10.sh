cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in "" "TPA_L2_FETCH=32" "TPA_L2_FETCH=64" "TPA_L2_FETCH=128"; do
  echo "== $v"; env $v TPA_DEBUG=1 python tools/ab_pre.py c5 2>&1 | grep -E "L2 fetch|spmv" | tail -2
  env $v python tools/ab_pre.py c4 2>&1 | tail -1
  env $v python tools/ab_pre.py c2 2>&1 | tail -1
  env $v python tools/ab_time.py c2 32 2>&1 | grep "ms/batch"
done
