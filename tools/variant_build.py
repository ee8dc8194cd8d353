"""Build A/B variants of libneob200.so that differ only in -D defines of
csrc/tbe_bucket.cu (the other objects are reused from the default build).
Usage: python tools/variant_build.py NAME DEF=VAL [DEF=VAL ...]
Output: abv/libneob200_NAME.so (select with NEO_B200_LIB=...)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2104_05158_b200 import _build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
_build.build()  # default objects up to date
out_dir = ROOT / "abv"
out_dir.mkdir(exist_ok=True)
obj = out_dir / f"tbe_bucket_{name}.o"
cc = _build.nvcc()
cmd = [cc, *_build.ARCH, *_build.FLAGS, *[f"-D{d}" for d in defs], "-I", str(_build.INCLUDE), "-I",
       str(_build.CSRC), "-c", str(_build.CSRC / "tbe_bucket.cu"), "-o", str(obj)]
subprocess.run(cmd, check=True)
objs = [p for p in sorted(_build.OBJ.glob("*.o")) if p.stem != "tbe_bucket"] + [obj]
lib = out_dir / f"libneob200_{name}.so"
subprocess.run([cc, *_build.ARCH, "-shared", "-o", str(lib), *map(str, objs)], check=True)
print(lib)
