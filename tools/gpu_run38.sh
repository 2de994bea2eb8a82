cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for v in default pdl default pdl; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  for c in c1 c2; do env $L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['value'],1), round(d['ms_per_step'],3))"; done
done
TPA_LIB=tools/bin/libtpa_pdl.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_partition.py tests/test_edge_cases.py -q -m gpu -x 2>&1 | tail -1
