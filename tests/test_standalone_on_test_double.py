"""CPU run of the standalone layer's GPU suites over the C-ABI test double
(tests/fake_native.py: host "device" memory, kernels by the C oracle), so
the pipeline, modes, chains, tiles and sharding host logic are exercised in
every CPU test run, not only on the B200.  Runs them in a subprocess with
TPG_FAKE_NATIVE=1 (tests/conftest.py installs the double)."""

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

SUITES = ["test_gpu_pipeline.py", "test_gpu_modes.py", "test_gpu_chain.py", "test_gpu_tile.py",
          "test_gpu_sharded.py", "test_gpu_golden.py"]


def test_gpu_suites_pass_on_the_test_double():
    env = dict(os.environ, TPG_FAKE_NATIVE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "-p", "no:cacheprovider", *[str(HERE / s) for s in SUITES]],
                       cwd=str(HERE.parent), env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
