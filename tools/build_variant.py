"""Experiment helper: build libios with extra -D flags into paper_2011_01302_b200/build/libios_<name>.so
(select it at run time with IOS_LIB=<path>). The product build is paper_2011_01302_b200/build.py.

  python tools/build_variant.py noprew -DIOS_NO_PREWEIGHTS
"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("_ios_build", os.path.join(ROOT, "paper_2011_01302_b200", "build.py"))
B = importlib.util.module_from_spec(spec)
spec.loader.exec_module(B)

name, defs = sys.argv[1], sys.argv[2:]
print(B.build(extra_defs=defs, out=os.path.join(B.HERE, "build", f"libios_{name}.so")))
