#!/usr/bin/env python
"""Build every native artefact in-tree (sm_100a only).

  fdgen/libfdgen.so                      input generators (host + device)
  oracle/liboracle.so                    CPU fp64 oracle (test infrastructure; gcc)
  paper_1501_06561_b200/libfd.so         the FD hot path: C ABI + sm_100a kernels

Usage: python build.py [--force] [target ...]
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)


def _glob(d, exts):
    out = []
    for root, _, files in os.walk(os.path.join(ROOT, d)):
        for f in files:
            if f.endswith(exts):
                out.append(os.path.join(root, f))
    return sorted(out)


def build_fdgen(force=False):
    out = os.path.join(ROOT, "fdgen", "libfdgen.so")
    srcs = _glob("fdgen/csrc", (".cu", ".h"))
    if force or _stale(out, srcs):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off", "-fmad=false",
              "-o", out, os.path.join(ROOT, "fdgen", "csrc", "fdgen.cu")])
    return out


def build_oracle(force=False):
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    srcs = _glob("oracle", (".c", ".h"))
    if force or _stale(out, srcs):
        _run(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-ffp-contract=off", "-pthread",
              "-o", out, os.path.join(ROOT, "oracle", "oracle.c"), "-lm"])
    return out


def build_libfd(force=False):
    """Each translation unit is compiled to an object in parallel (build/libfd/), then
    linked; a unit is recompiled when it, any header or the extra flags changed."""
    import concurrent.futures as cf
    pkg = os.path.join(ROOT, "paper_1501_06561_b200")
    out = os.path.join(pkg, "libfd.so")
    srcs = _glob("paper_1501_06561_b200/csrc", (".cu", ".cuh", ".cpp", ".h")) + _glob("include", (".h",))
    cu = [s for s in srcs if s.endswith((".cu", ".cpp"))]
    hdr = [s for s in srcs if not s.endswith((".cu", ".cpp"))]
    if not cu:
        return None
    extra = os.environ.get("FD_NVCC_EXTRA", "").split()   # e.g. -DFD_INV_ITERS=2 (A/B builds)
    stamp = out + ".flags"
    prev = open(stamp).read() if os.path.exists(stamp) else ""
    flags_changed = prev != " ".join(extra)
    objdir = os.path.join(ROOT, "build", "libfd")
    os.makedirs(objdir, exist_ok=True)
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v" if os.environ.get("FD_PTXAS_V") else "-O3",
              "-I", os.path.join(ROOT, "include"), "-I", os.path.join(pkg, "csrc"), *extra]
    objs, todo = [], []
    for src in cu:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or flags_changed or _stale(obj, [src] + hdr):
            todo.append((src, obj))
    with cf.ThreadPoolExecutor(max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        list(ex.map(lambda so: _run(common + ["-c", "-o", so[1], so[0]]), todo))
    if todo or _stale(out, objs):
        _run([NVCC, *ARCH, "-shared", "-o", out, *objs])
        with open(stamp, "w") as f:
            f.write(" ".join(extra))
    return out


TARGETS = {"fdgen": build_fdgen, "oracle": build_oracle, "libfd": build_libfd}


def build_all(force=False, targets=None):
    outs = []
    for name in targets or TARGETS:
        outs.append(TARGETS[name](force))
    return outs


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    build_all(force="--force" in sys.argv, targets=args or None)
