"""Build oracle/libspin_oracle.so (the C++ oracle) — TEST INFRASTRUCTURE ONLY.

Called by __graft_entry__.build() (building the checker is not using it) and, if the
library is missing, by oracle/spin_oracle_cpp.py on first use.  Plain g++ -O2, no FMA
contraction (the stage-1 error bounds assume one rounding per operation).
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "spin_oracle.cpp")
OUT = os.path.join(HERE, "libspin_oracle.so")
CMD = ["g++", "-O2", "-march=x86-64-v3", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
       "-pthread", "-Wall", "-o", OUT + ".tmp", SRC]


def build(force: bool = False) -> str:
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= os.path.getmtime(SRC):
        return OUT
    r = subprocess.run(CMD, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + " ".join(CMD) + "\n" + r.stdout)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True))
