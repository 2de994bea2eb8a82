for v in "" "TPA_MV_CARVEOUT=25" "TPA_MV_CARVEOUT=40" "TPA_MV_CARVEOUT=50" "TPA_MV_CARVEOUT=60" "TPA_MV_CARVEOUT=100"; do
echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "spmv"; done
