"""Build recipe for the C oracle (test infrastructure).

The reference is Python + numba, so there is no C/C++ reference to compile into
oracle/_ref; the oracle is a C restatement (mpm_oracle.c) pinned against arrays dumped
from the reference (tests/golden/).  -ffp-contract=off keeps products and sums rounded
separately, as in the reference's non-fastmath numba kernels.
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mpm_oracle.c")
OUT = os.path.join(HERE, "libmpm_oracle.so")


def build(force: bool = False) -> str:
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= os.path.getmtime(SRC):
        return OUT
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-o", OUT, SRC, "-lm"]
    subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    print(build(force=True))
