"""Build libspin.so in-tree for sm_100a (called by __graft_entry__.build()).

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; cudart linked
statically so the library does not depend on the process's libcudart.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libspin.so")
BUILD = os.path.join(HERE, "..", "build", "spin")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]
# (source, extra defines, object name): the persistent kernel's 112 instantiations are
# split over twelve translation units (one per (mode, support placement, dealer) triple)
UNITS = [("spin_kernels.cu", (), "spin_kernels"), ("spin_api.cpp", (), "spin_api"),
         ("spin_io.cpp", (), "spin_io")] + [
    ("spin_inst.cu", (f"-DINST_MODE={m}", f"-DINST_SUP={u}", f"-DINST_DEAL={d}"), f"spin_inst_{m}_{u}_{d}")
    for m in (0, 1) for u in (0, 1, 2) for d in (0, 1)]
SOURCES = [u[0] for u in UNITS]


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout)
    return r.stdout


def _stale(objs):
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "spin.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defs: tuple = ()) -> str:
    """Build libspin.so (or, for A/B measurements, a variant with -D`defs` at `out`)."""
    global OUT
    if out:
        OUT = os.path.abspath(out)
        os.makedirs(os.path.dirname(OUT), exist_ok=True)
    build_dir = BUILD if not defs else BUILD + "_" + "_".join(d.strip("-D").replace("=", "") for d in defs)
    os.makedirs(build_dir, exist_ok=True)
    objs = [os.path.join(build_dir, u[2] + ".o") for u in UNITS]
    if not force and not defs and not _stale(objs):
        return OUT
    def comp(unit, obj):
        src, udefs, _ = unit
        extra = ["-Xptxas", "-v"] if (verbose and src.endswith(".cu")) else []
        cmd = [NVCC, *ARCH, *FLAGS, *defs, *udefs, *extra, "-I", os.path.join(HERE, "..", "include"),
               "-c", os.path.join(CSRC, src), "-o", obj]
        return _run(cmd)
    with ThreadPoolExecutor(len(UNITS)) as ex:
        logs = list(ex.map(comp, UNITS, objs))
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", OUT + ".tmp", *objs])
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print("".join(logs))
    return OUT


if __name__ == "__main__":
    out = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")), None)
    defs = tuple(a for a in sys.argv if a.startswith("-D"))
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=out, defs=defs))
