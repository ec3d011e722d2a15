"""In-tree build of libcgb200.so for sm_100a (no JIT cache, travels with the repo)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "cgb200.cu")
DEPS = [SRC, os.path.join(HERE, "csrc", "cgb_device.cuh"),
        os.path.join(HERE, "csrc", "cgb_shard.cuh"),
        os.path.join(HERE, "csrc", "cgb_shard_kernel.cuh"),
        os.path.join(os.path.dirname(HERE), "include", "cgb200.h")]
OUT = os.path.join(HERE, "lib", "libcgb200.so")

NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


# translation units compiled in parallel (see the CGB_TU_* flags in cgb200.cu)
UNITS = ["CGB_TU_HOST", "CGB_TU_SCS0", "CGB_TU_SCS1", "CGB_TU_SCS2", "CGB_TU_CG", "CGB_TU_INNER",
         "CGB_TU_MISC", "CGB_TU_SHARD"]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    objdir = os.path.join(os.path.dirname(OUT), "obj")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]
    procs = []
    for unit in UNITS:
        obj = os.path.join(objdir, unit.lower() + ".o")
        cmd = [nvcc(), *cflags, "-DCGB_SPLIT", f"-D{unit}=1", "-c", "-o", obj, SRC]
        procs.append((unit, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                  stderr=subprocess.PIPE, text=True)))
    objs, logs = [], []
    for unit, obj, pr in procs:
        out, err = pr.communicate()
        logs.append(err)
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed on {unit} ({pr.returncode}):\n{err[-4000:]}")
        objs.append(obj)
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
            "-fPIC", "-o", OUT + ".tmp", *objs]
    proc = subprocess.run(link, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({proc.returncode}):\n{proc.stderr[-4000:]}")
    if verbose:
        print("\n".join(logs))
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
