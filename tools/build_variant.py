"""Experiment helper: build libios with extra -D flags into paper_2011_01302_b200/build/libios_<name>.so
(select it at run time with IOS_LIB=<path>). The product build is paper_2011_01302_b200/build.py.

  python tools/build_variant.py nozero -DIOS_EXP_NOZERO
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_01302_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
bdir = os.path.join(B.HERE, "build", name)
os.makedirs(bdir, exist_ok=True)
objs = []
for src in B.SOURCES:
    obj = os.path.join(bdir, src + ".o")
    subprocess.run([B.NVCC, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    objs.append(obj)
out = os.path.join(B.HERE, "build", f"libios_{name}.so")
subprocess.run([B.NVCC, *B.FLAGS, "-shared", "-o", out, *objs], check=True)
print(out)
