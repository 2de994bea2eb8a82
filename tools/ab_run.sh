set -x
python tools/ab_time.py c2 32 2>&1 | grep -v Warn
TPA_MM5_RB=4 python tools/ab_time.py c2 32 2>&1 | grep -v Warn
TPA_LIB=tools/bin/libtpa_minb10.so python tools/ab_time.py c2 32 2>&1 | grep -v Warn
TPA_LIB=tools/bin/libtpa_minb10.so TPA_MM5_RB=4 python tools/ab_time.py c2 32 2>&1 | grep -v Warn
python tools/ab_time.py c3 64 2>&1 | grep -v Warn
TPA_MM5_RB=4 python tools/ab_time.py c3 64 2>&1 | grep -v Warn
TPA_LIB=tools/bin/libtpa_minb6.so python tools/ab_time.py c3 64 2>&1 | grep -v Warn
