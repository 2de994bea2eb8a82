python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
python tools/ab_time.py c2 32 2>&1 | grep -E "sweep |ms/batch"
python tools/ab_time.py c3 64 2>&1 | grep -E "ms/batch"
