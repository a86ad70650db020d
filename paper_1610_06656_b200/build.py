"""Build libsmp.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_1610_06656_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsmp.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps.append(os.path.join(ROOT, "include", "smp.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _fresh(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return False
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    hdrs.append(os.path.join(ROOT, "include", "smp.h"))
    t = os.path.getmtime(obj)
    return all(os.path.getmtime(d) < t for d in [src, *hdrs])


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None, only=()) -> str:
    """Compile csrc/*.cu (in parallel) and link libsmp.so.  `defines` and
    `out` produce tuning variants (e.g. libsmp_x4p3.so) next to the default."""
    out = out or LIB
    if not force and out == LIB and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    tag = os.path.basename(out).replace(".so", "")
    objdir = os.path.join(PKG, "build", tag)
    os.makedirs(objdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    procs = []
    default_objs = os.path.join(PKG, "build", "libsmp")
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        if only and os.path.basename(src) not in only:
            # tuning variant: reuse the default build's object for this source
            ref = os.path.join(default_objs, os.path.basename(obj))
            if not os.path.exists(ref):
                raise RuntimeError(f"variant build needs the default object {ref}")
            procs.append((src, ref, None))
            continue
        if not force and not dflags and _fresh(src, obj):
            procs.append((src, obj, None))  # incremental: object newer than its inputs
            continue
        cmd = [nvcc, *NVCC_FLAGS, *dflags, "-c", src, "-o", obj, "-I", os.path.join(ROOT, "include")]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                                 text=True)))
    objs = []
    for src, obj, pr in procs:
        if pr is None:
            objs.append(obj)
            continue
        so, se = pr.communicate()
        if pr.returncode != 0:
            sys.stderr.write(so + se)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(se)
        objs.append(obj)
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out + ".tmp", *objs,
           "-Xcompiler", "-fPIC"]
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    defs = [a[2:] for a in args if a.startswith("-D")]
    outs = [a for a in sys.argv[1:] if a.startswith("--out=")]
    only = [a[7:] for a in sys.argv[1:] if a.startswith("--only=")]
    print(build(force="--force" in sys.argv or bool(defs), verbose="--quiet" not in sys.argv,
                defines=defs, out=os.path.join(PKG, outs[0][6:]) if outs else None,
                only=tuple(x for o in only for x in o.split(","))))
