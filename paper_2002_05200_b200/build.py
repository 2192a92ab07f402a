"""Build the sm_100a C-ABI library in-tree (nvcc, no JIT, no torch extension)."""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblogan_xdrop.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    *ARCH,
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
    "-I", CSRC,
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(ROOT, "include", "logan_xdrop.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Build the library (``out`` / ``defines`` build an experimental variant)."""
    target = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    tmp = target + ".tmp"
    # one translation unit per format (logan_fmt_*.cu) plus the C ABI, compiled in
    # parallel (each is a few hundred kernel instantiations), then linked
    units = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    objdir = tempfile.mkdtemp(prefix="logan_build_")
    objs, procs = [], []
    for u in units:
        o = os.path.join(objdir, os.path.basename(u) + ".o")
        objs.append(o)
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", "-o", o, u]
        procs.append((u, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    logs, failed = [], []
    for u, pr in procs:
        out_, err = pr.communicate()
        logs.append(f"==== {os.path.basename(u)}\n{err}")
        if pr.returncode != 0:
            failed.append(u)
            sys.stderr.write(out_ + err)
    if failed:
        raise RuntimeError(f"nvcc failed building liblogan_xdrop.so ({', '.join(map(os.path.basename, failed))})")
    res = subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking liblogan_xdrop.so")
    shutil.rmtree(objdir, ignore_errors=True)
    if out is None:
        with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    if verbose:
        sys.stderr.write("\n".join(logs))
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
