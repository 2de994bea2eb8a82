python tools/ab_time.py c2 64 2>&1 | grep -E "sweep |ms/batch"
python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
