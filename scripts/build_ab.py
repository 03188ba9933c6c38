"""Build libtidepool_gpu.so of another git revision for same-box A/B runs
(box-to-box variance is several %, larger than the effects being measured).

usage: python scripts/build_ab.py <rev> <name>
  -> ab_libs/lib_<name>.so  (select it with TIDEPOOL_GPU_LIB=ab_libs/lib_<name>.so)
"""
import concurrent.futures as cf
import os
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1810_08723_b200 import build as B  # noqa: E402


def main(rev, name):
    out = ROOT / "ab_libs"
    out.mkdir(exist_ok=True)
    tmp = Path(tempfile.mkdtemp(prefix=f"ab_{name}_"))
    arch = subprocess.run(["git", "-C", str(ROOT), "archive", rev, "paper_1810_08723_b200/csrc",
                           "include"], check=True, capture_output=True).stdout
    subprocess.run(["tar", "-x", "-C", str(tmp)], input=arch, check=True)
    csrc = tmp / "paper_1810_08723_b200" / "csrc"
    srcs = sorted(csrc.glob("*.cu"))

    def comp(src):
        obj = tmp / (src.stem + ".o")
        flags = [f if not f.startswith("-I") else f"-I{tmp / 'include'}" for f in B.COMMON]
        cmd = [B.NVCC, *B.ARCH, *flags, "-c", str(src), "-o", str(obj)]
        if src.name.startswith(B.NO_FMA_PREFIX):
            cmd.insert(1, "-fmad=false")
        subprocess.run(cmd, check=True)
        return obj
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 8) as ex:
        objs = list(ex.map(comp, srcs))
    lib = out / f"lib_{name}.so"
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart",
                    "-ldl", "-lcuda"], check=True)
    print(lib)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
