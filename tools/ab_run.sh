for v in "" "TPA_MM5_CARVEOUT=58" "TPA_MM5_CARVEOUT=45" "TPA_MM5_CARVEOUT=100"; do
echo "== $v"; env $v python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
done
