python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/ab_time.py c2 32 2>&1 | grep -E "spmv|ms/batch"
