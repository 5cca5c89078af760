"""Build an A/B variant of libposit_b200.so with extra -D flags (same sources,
same nvcc flags as paper_2401_14117_b200/build.py) into
paper_2401_14117_b200/ab/libposit_<name>.so; load it with POSIT_LIB_PATH.

    python tools/build_variant.py tab64 -DPGD_TAB32=0
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_14117_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(B.HERE, "ab"), exist_ok=True)
out = os.path.join(B.HERE, "ab", f"libposit_{name}.so")
subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-I", B.INCLUDE, "-o", out, *B.sources()], check=True)
print(out)
