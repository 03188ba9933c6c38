"""Build recipe for the CPU oracle (test infrastructure, not product).

Compiles oracle/tp_oracle.c into oracle/_build/libtp_oracle.so with gcc
(OpenMP for the multi-core CPU baseline).  The reference implementation is
pure Python (pkg/src/tidepool), so there is no compiled reference to put in
oracle/_ref; the Python reference is used in this container only, to
generate the golden vectors under tests/golden/.
"""

from __future__ import annotations

import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "tp_oracle.c"
OUT = HERE / "_build" / "libtp_oracle.so"


def build(verbose: bool = False) -> Path:
    OUT.parent.mkdir(exist_ok=True)
    deps = [SRC, HERE.parent / "include" / "tidepool_gpu.h"]
    if OUT.exists() and all(d.stat().st_mtime <= OUT.stat().st_mtime for d in deps):
        return OUT
    # -ffp-contract=off: every + - * is a separately rounded double op, as in
    # CPython; -fno-fast-math semantics are the default.
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-builtin", "-o", str(OUT), str(SRC), "-lm"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True))
