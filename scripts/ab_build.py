"""Build variant libraries for A/B timing (dev tool): each variant is the
current csrc/ with some files replaced by their version at a git revision.
usage: python scripts/ab_build.py NAME REV [-DMACRO=V ...] file [file ...]
  -> build/ab/NAME/libasyncspade.so"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07486_b200 import build as B  # noqa: E402

name, rev = sys.argv[1], sys.argv[2]
defines = [a for a in sys.argv[3:] if a.startswith("-D")]
files = [a for a in sys.argv[3:] if not a.startswith("-D")]
out = os.path.join(ROOT, "build", "ab", name)
src = os.path.join(out, "csrc")
shutil.rmtree(out, ignore_errors=True)
shutil.copytree(B.CSRC, src)
for f in files:
    blob = subprocess.run(["git", "show", f"{rev}:paper_2510_07486_b200/csrc/{f}"], cwd=ROOT,
                          capture_output=True, text=True, check=True).stdout
    open(os.path.join(src, f), "w").write(blob)
objs = []
flags = [x if x != B.CSRC else src for x in B.NVCC_FLAGS]
for f in B.PRODUCT_SOURCES:
    o = os.path.join(out, f + ".o")
    subprocess.run([B._nvcc(), *B.ARCH, *flags, *defines, "-c", os.path.join(src, f), "-o", o], check=True,
                   capture_output=True)
    objs.append(o)
lib = os.path.join(out, "libasyncspade.so")
subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs], check=True)
print(lib)
