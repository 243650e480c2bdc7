"""Build the sm_100a C-ABI library in-tree: ``python -m paper_2504_13339_b200.build``."""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

CSRC = Path(__file__).resolve().parent / "csrc"


def build(jobs: int = 4, verbose: bool = False) -> Path:
    out = subprocess.run(["make", f"-j{jobs}", "-C", str(CSRC)], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"nvcc build failed:\n{out.stdout[-4000:]}\n{out.stderr[-8000:]}")
    if verbose:
        print(out.stdout[-2000:])
    from ._lib import LIB_PATH

    return LIB_PATH


if __name__ == "__main__":
    print(build(jobs=os.cpu_count() or 4))
