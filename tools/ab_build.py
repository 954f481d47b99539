"""Build a variant of the native library into _ab/<name>.so with extra nvcc
flags (A/B kernel experiments; load it with ATA_LIB_PATH=_ab/<name>.so).

  python tools/ab_build.py NAME [-DMACRO ...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2110_13042_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = Path(__file__).resolve().parent.parent / "_ab"
out.mkdir(exist_ok=True)
B.LIBDIR = out / ("obj_" + name)
B.LIB = out / (name + ".so")
B.NVCC_FLAGS = B.NVCC_FLAGS + extra
print(B.build(force=True))
