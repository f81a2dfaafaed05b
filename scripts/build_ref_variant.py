"""Builds librelief_b200.so from the csrc/ of a git revision into ab/NAME (A/B baselines).

Usage: python scripts/build_ref_variant.py REV NAME [-DFOO=1 ...]
REV = WORKTREE builds the working tree's sources (with the given defines).
"""
import subprocess
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2204_12876_b200 import build as b  # noqa: E402

rev, name, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
tmp = Path(tempfile.mkdtemp())
for sub in ("paper_2204_12876_b200/csrc", "include"):
    (tmp / sub).mkdir(parents=True)
    if rev == "WORKTREE":
        for f in (b.ROOT / sub).iterdir():
            if f.is_file():
                (tmp / sub / f.name).write_bytes(f.read_bytes())
        continue
    files = subprocess.run(["git", "-C", str(b.ROOT), "ls-tree", "--name-only", f"{rev}:{sub}"],
                           capture_output=True, text=True, check=True).stdout.split()
    for f in files:
        data = subprocess.run(["git", "-C", str(b.ROOT), "show", f"{rev}:{sub}/{f}"], capture_output=True,
                              check=True).stdout
        (tmp / sub / f).write_bytes(data)
out = b.ROOT / "ab" / name
b.CSRC = tmp / "paper_2204_12876_b200" / "csrc"
b.OBJ = out / "obj"
b.LIB_DIR = out
b.LIB = out / "librelief_b200.so"
b.NVCC_FLAGS = [f.replace(str(b.ROOT / "include"), str(tmp / "include")).replace(str(b.PKG / "csrc"), str(b.CSRC))
                for f in b.NVCC_FLAGS] + defs
b.CXX_FLAGS = [f.replace(str(b.ROOT / "include"), str(tmp / "include")).replace(str(b.PKG / "csrc"), str(b.CSRC))
               for f in b.CXX_FLAGS]
print(b.build(force=True))
