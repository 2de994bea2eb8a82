"""A/B builds of libtpa_gpu.so with compile-time knobs (experiments only).

    python tools/ab_variants.py NAME "-DKNOB=1 -DOTHER=0" [NAME "..."]...

Each variant is a copy of the package under tools/bin/NAME/ (git-ignored; it
travels to the GPU box with gpurun) built with the extra nvcc flags; run a
script against it with PYTHONPATH=tools/bin/NAME.  The product library is not
touched.
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1708_02574_b200")
sys.path.insert(0, PKG)
import build as B  # noqa: E402


def make(name, flags):
    dst = os.path.join(ROOT, "tools", "bin", name, "paper_1708_02574_b200")
    os.makedirs(dst, exist_ok=True)
    for f in os.listdir(PKG):
        if f.endswith(".py"):
            shutil.copy(os.path.join(PKG, f), dst)
    lib = os.path.join(dst, "libtpa_gpu.so")
    cmd = [shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc", *B.NVCC_FLAGS, *flags.split(), "-shared",
           "-I", B.INCLUDE, "-I", B.CSRC, "-o", lib, *B.sources(), *B.LIBS]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stderr[-3000:])
        raise SystemExit(f"variant {name} failed")
    print(name, flags, "->", lib)


if __name__ == "__main__":
    args = sys.argv[1:]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(4) as ex:
        list(ex.map(lambda p: make(*p), zip(args[0::2], args[1::2])))
