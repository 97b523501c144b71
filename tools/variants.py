"""Build variant libraries (same sources, different tuning macros) under build_variants/.

    python tools/variants.py NAME=DEF1,DEF2 ...    e.g.  ub2_b3=ONEDF_FWD_UB=2,ONEDF_FWD_MINB=3
Each lands in build_variants/NAME/libonedf.so; select one with ONEDF_LIB=... (tools only).
"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2501_14577_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
for arg in sys.argv[1:]:
    name, defs = arg.split("=", 1)
    d = os.path.join(ROOT, "build_variants", name)
    os.makedirs(d, exist_ok=True)
    print(b.build(defines=[x for x in defs.split(",") if x], lib=os.path.join(d, "libonedf.so"), objdir=d))
