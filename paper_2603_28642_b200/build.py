"""Build librowsplit_b200.so in-tree (nvcc -gencode arch=compute_100a,code=sm_100a)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build(jobs: int = 4) -> str:
    subprocess.run(["make", "-s", f"-j{jobs}", "-C", os.path.join(HERE, "csrc")], check=True)
    from ._lib import LIB_PATH
    return LIB_PATH


if __name__ == "__main__":
    print(build())
