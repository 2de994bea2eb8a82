#!/bin/bash
# The driver's round-end sequence on one box: -m gpu tests, smoke, the reference
# arm, the default bench line.  Logs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
( time timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --durations=8 ) > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/final_pytest_gpu.log
( time python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/final_smoke.log 2>&1; echo "smoke rc $?"; tail -4 gpurun_out/final_smoke.log
( time python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc $?"; tail -3 gpurun_out/final_ref.err
( time python bench.py --steps 20 --warmup 5 ) > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc $?"; tail -3 gpurun_out/final_bench.err
python - <<'PY'
import json
for f in ("gpurun_out/final_ref.json", "gpurun_out/final_bench.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("frac"),
              (d.get("roofline") or {}).get("l2_bound"), d.get("clocks"))
    except Exception as e:
        print(f, "unreadable", e)
PY
