python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
ncu --set full --clock-control none --import-source on -k regex:"k_mm_fused" -s 0 -c 2 -o gpurun_out/sparse_full2 python tools/profile_step.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 60 --csv --log-file gpurun_out/ll_def.csv python tools/profile_step.py --batches 3 > /dev/null 2>&1
