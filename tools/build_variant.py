"""Builds an A/B variant of libtpa_gpu.so with extra -D flags into tools/bin/:
python tools/build_variant.py NAME -DFOO=1 ...   (then TPA_LIB=tools/bin/libtpa_NAME.so)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_1708_02574_b200"))
import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "tools", "bin"), exist_ok=True)
out = os.path.join(ROOT, "tools", "bin", f"libtpa_{name}.so")
cmd = ["nvcc", *B.NVCC_FLAGS, *extra, "-shared", "-I", B.INCLUDE, "-I", B.CSRC, "-o", out, *B.sources(), *B.LIBS]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
for line in r.stderr.splitlines():
    if "k_mm_fused" in line or ("registers" in line and "spill" in line):
        pass
print(out)
