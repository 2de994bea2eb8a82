python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" "TPA_PUSH_SWEEPS=0" "TPA_PUSH_DIV=4" "TPA_PUSH_SWEEPS=1"; do
  echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
done
python tools/ab_time.py c3 64 2>&1 | grep -E "sweep |ms/batch"
