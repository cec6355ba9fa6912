"""Build a tuning variant of libsunbw.so under build/<name>/ with extra
-D defines for fused.cu only (the other objects are the default build's).
Usage: python tools/build_variant.py NAME DEFINE [DEFINE ...]"""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_12984_b200 import _build  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
_build.build()
obj = os.path.join(ROOT, "build", name, "obj")
os.makedirs(obj, exist_ok=True)
for f in os.listdir(_build.OBJDIR):
    if f != "fused.o":
        shutil.copy2(os.path.join(_build.OBJDIR, f), os.path.join(obj, f))
fo = os.path.join(obj, "fused.o")
if os.path.exists(fo):
    os.remove(fo)
print(_build.build(defines=defines, out=os.path.join(ROOT, "build", name, "libsunbw.so")))
