"""Builds an A/B variant of librelief_b200.so with extra nvcc defines.

Usage: python scripts/build_variant.py NAME -DFOO=1 ...
Output: ab/NAME/librelief_b200.so (git-ignored; travels with gpurun). Load it
with RELIEF_B200_LIB=ab/NAME/librelief_b200.so.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2204_12876_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = b.ROOT / "ab" / name
b.OBJ = out / "obj"
b.LIB_DIR = out
b.LIB = out / "librelief_b200.so"
b.NVCC_FLAGS = b.NVCC_FLAGS + defs
print(b.build(force=True))
