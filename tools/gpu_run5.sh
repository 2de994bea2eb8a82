cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in default al uh aluh default; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== c2/32 $v"; env $L python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
  echo "== c2/16 $v"; env $L python tools/ab_time.py c2 16 2>&1 | grep -E "ms/batch"
done
for v in default aluh; do
  if [ $v = default ]; then L=""; else L="TPA_LIB=tools/bin/libtpa_$v.so"; fi
  echo "== c3/64 $v"; env $L python tools/ab_time.py c3 64 2>&1 | grep -E "ms/batch"
done
echo "== c2/16 RB16"; TPA_MM5_RB=16 python tools/ab_time.py c2 16 2>&1 | grep -E "sweep |ms/batch"
python tools/profile_step.py --config c5 --batch 16 --batches 1 > gpurun_out/c5_plain.log 2>&1; echo "c5 plain rc $?"
ncu --set full --clock-control none --import-source on -k regex:"k_step_spmv2" -s 20 -c 1 -o gpurun_out/c5_spmv python tools/profile_step.py --config c5 --batch 16 --batches 1 > gpurun_out/c5_ncu1.log 2>&1; echo "ncu spmv rc $?"
ncu --set full --clock-control none --import-source on -k regex:"k_mm_fused" -s 1 -c 2 -o gpurun_out/c5_spmm python tools/profile_step.py --config c5 --batch 16 --batches 1 > gpurun_out/c5_ncu2.log 2>&1; echo "ncu spmm rc $?"
