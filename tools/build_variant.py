"""Build libcgb200.so with extra -D flags into lib/variants/<name>/ (for
A/B timing with CGB200_LIB=<path>; development aid).

usage: python tools/build_variant.py <name> -DFOO=1 [-DBAR=2 ...]
"""
import os
import subprocess
import sys

sys.path.insert(0, ".")
from paper_1609_03488_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(os.path.dirname(B.OUT), "variants", name)
os.makedirs(out_dir, exist_ok=True)
cflags = [f for f in B.NVCC_FLAGS if f != "-shared"]
procs = []
for unit in B.UNITS:
    obj = os.path.join(out_dir, unit.lower() + ".o")
    cmd = [B.nvcc(), *cflags, *defs, "-DCGB_SPLIT", f"-D{unit}=1", "-c", "-o", obj, B.SRC]
    procs.append((obj, subprocess.Popen(cmd, stderr=subprocess.PIPE, stdout=subprocess.PIPE,
                                        text=True)))
objs = []
for obj, pr in procs:
    _, err = pr.communicate()
    if pr.returncode:
        sys.exit(err[-3000:])
    objs.append(obj)
lib = os.path.join(out_dir, "libcgb200.so")
subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                "-fPIC", "-o", lib, *objs], check=True)
for o in objs:
    os.remove(o)
print(lib)
