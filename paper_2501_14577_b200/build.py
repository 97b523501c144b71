"""Build libonedf.so (all CUDA kernels + the C ABI) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import concurrent.futures
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libonedf.so")
OBJDIR = os.path.join(PKG, "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
         "--fmad=true", "-I", INCLUDE, "-I", CSRC]
SOURCES = ["fwd_inst.cu", "bwd_inst.cu", "encode.cu", "sort.cu", "mean.cu", "fwd.cu", "bwd.cu", "csr.cu",
           "proj.cu", "workload.cu", "abi.cu"]
# Compilation units: (object, source, unit defines).  The kernel-template instantiation sources are
# compiled once per unit (value storage type x register rows / d_k pair) so the instantiations build in parallel;
# heaviest first.
UNITS = ([(f"fwd_{n}_r{r}", "fwd_inst.cu", (f"ONEDF_INST_TV={tv}", f"ONEDF_INST_TV_{tv.upper()}", f"ONEDF_INST_R={r}"))
          for r in (8, 4, 2, 1) for n, tv in (("f32", "float"), ("bf16", "bf16"))]
         + [(f"bwd_{n}_dk{a}{b}", "bwd_inst.cu", (f"ONEDF_INST_TV={tv}", f"ONEDF_INST_DK_A={a}", f"ONEDF_INST_DK_B={b}"))
            for n, tv in (("f32", "float"), ("bf16", "bf16")) for a, b in ((1, 2), (3, 4), (5, 6), (7, 8))]
         + [(src[:-3], src, ()) for src in SOURCES if not src.endswith("_inst.cu")])


def _stamp(files, defines) -> str:
    """Content hash of the sources, headers and flags a library is built from."""
    h = hashlib.sha256()
    for f in sorted(files, key=lambda x: os.path.relpath(x, ROOT)):
        with open(f, "rb") as fh:      # repo-relative names: the same stamp wherever the checkout lives
            h.update(os.path.relpath(f, ROOT).encode() + b"\0" + fh.read())
    h.update(" ".join(ARCH + FLAGS + list(defines)).encode())
    return h.hexdigest()


def _read(path: str):
    try:
        with open(path) as f:
            return f.read()
    except OSError:
        return None


def _headers():
    hs = [os.path.join(INCLUDE, "onedf.h")]
    hs += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB, objdir: str = OBJDIR,
          define_srcs=None) -> str:
    """defines/lib/objdir: variant builds for tools/ experiments (the product is the default);
    define_srcs: apply the defines only to the units of these sources (others as in the product)."""
    os.makedirs(objdir, exist_ok=True)
    hdrs = _headers()
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    stamp = _stamp(srcs + hdrs, defines)
    if not force and not defines and _read(lib + ".stamp") == stamp and os.path.exists(lib):
        return lib          # built from exactly these sources and flags (objects need not be present)
    jobs = []
    for obj, src, udefs in UNITS:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, obj + ".o")
        # per-object content stamp (source + every header + flags + defines): an object is reused
        # only if it was built from exactly these inputs, whatever the files' mtimes say
        defs = tuple(defines) if define_srcs is None or src in define_srcs else ()
        ostamp = _stamp([s] + hdrs, defs + tuple(udefs))
        if force or not os.path.exists(o) or _read(o + ".stamp") != ostamp:
            cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defs + tuple(udefs)], "-c", s, "-o", o]
            if verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append((cmd, o, ostamp))

    def run(job):
        cmd, o, ostamp = job
        if os.path.exists(o + ".stamp"):
            os.remove(o + ".stamp")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {o}:\n{r.stderr}")
        with open(o + ".stamp", "w") as f:
            f.write(ostamp)
        return r.stderr

    with concurrent.futures.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for log in ex.map(run, jobs):
            if verbose and log:
                sys.stderr.write(log)
    objs = [os.path.join(objdir, obj + ".o") for obj, _, _ in UNITS]
    if force or jobs or not os.path.exists(lib) or _read(lib + ".stamp") != stamp:
        cmd = [NVCC, *ARCH, "-shared", "-o", lib + ".tmp", *objs, "-lcudart"]
        subprocess.run(cmd, check=True)
        os.replace(lib + ".tmp", lib)
    if not defines and _stamp(srcs + hdrs, defines) == stamp:   # sources unchanged while compiling
        with open(lib + ".stamp", "w") as f:
            f.write(stamp)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
