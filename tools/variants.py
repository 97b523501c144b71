"""Build variant libraries (same sources, different tuning macros) under build_variants/.

    python tools/variants.py [--src fwd.cu,bwd.cu] NAME=DEF1,DEF2 ...
        e.g.  python tools/variants.py --src fwd_inst.cu sub2=ONEDF_FWD_SUB=2
              (backward kernel macros: --src bwd_inst.cu)
Each lands in build_variants/NAME/libonedf.so; select one with ONEDF_LIB=... (tools only).
With --src only the compilation units of those sources are recompiled with the defines; the
other objects are copied from the product build (paper_2501_14577_b200/build/), which must be
current.
"""
import argparse
import importlib.util
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2501_14577_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)

ap = argparse.ArgumentParser()
ap.add_argument("--src", default="")
ap.add_argument("variants", nargs="+")
a = ap.parse_args()
only = [s for s in a.src.split(",") if s]
for arg in a.variants:
    name, defs = arg.split("=", 1)
    d = os.path.join(ROOT, "build_variants", name)
    os.makedirs(d, exist_ok=True)
    if only:
        for obj, src, _ in b.UNITS:
            o = obj + ".o"
            if src in only:
                if os.path.exists(os.path.join(d, o)):
                    os.remove(os.path.join(d, o))
            else:
                shutil.copy2(os.path.join(b.OBJDIR, o), os.path.join(d, o))
                shutil.copy2(os.path.join(b.OBJDIR, o + ".stamp"), os.path.join(d, o + ".stamp"))
    print(b.build(defines=[x for x in defs.split(",") if x], lib=os.path.join(d, "libonedf.so"), objdir=d,
                  define_srcs=only or None))
