"""Run the reference's own pytest suite with gpu0 as the default device.

The reference tests are reference SOURCE, so they are not in this repo:
stage them once with `python scripts/run_reference_suite.py --stage`
(copies /root/reference/pkg/tests into baseline/_ref_tests, git-ignored,
travels to the GPU box with gpurun like baseline/_ref).  Then

    python scripts/run_reference_suite.py            # on a B200
    python scripts/run_reference_suite.py --fake     # CPU, C-oracle test double

Extra arguments are passed to pytest.  Exit code = pytest's.
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
STAGED = ROOT / "baseline" / "_ref_tests"
SOURCE = Path("/root/reference/pkg/tests")


def main(argv):
    if "--stage" in argv:
        if STAGED.exists():
            shutil.rmtree(STAGED)
        shutil.copytree(SOURCE, STAGED, ignore=shutil.ignore_patterns("__pycache__"))
        print(f"staged {SOURCE} -> {STAGED}")
        return 0
    env = dict(os.environ)
    if "--fake" in argv:
        env["TPG_REFSUITE_FAKE"] = "1"
        argv = [a for a in argv if a != "--fake"]
    tests = STAGED if STAGED.exists() else SOURCE
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests"), str(ROOT),
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", str(tests), "-p", "refsuite_gpu", "-p",
           "no:cacheprovider", "-q", "-o", "addopts=", "--rootdir", str(tests), *argv]
    return subprocess.call(cmd, env=env, cwd=str(ROOT))


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
