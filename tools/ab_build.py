#!/usr/bin/env python
"""Build libmg.so from a git revision's csrc (or the working tree) into _ab/<tag>/ for
A/B timing on the GPU box (tools/stage_breakdown.py --lib _ab/<tag>/libmg.so).

  python tools/ab_build.py <tag> [<rev>]      # rev omitted: the working tree
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    tag = sys.argv[1]
    rev = sys.argv[2] if len(sys.argv) > 2 else None
    from paper_2512_08555_b200 import build as B
    out = os.path.join(ROOT, "_ab", tag)
    src = os.path.join(out, "pkg", "csrc")  # csrc includes "../../include/mg.h"
    inc = os.path.join(out, "include")
    os.makedirs(src, exist_ok=True)
    os.makedirs(inc, exist_ok=True)
    files = B.SOURCES + ["mg_internal.h"]
    for f in files:
        p = "paper_2512_08555_b200/csrc/" + f
        if rev:
            data = subprocess.run(["git", "show", f"{rev}:{p}"], cwd=ROOT, check=True, capture_output=True).stdout
            open(os.path.join(src, f), "wb").write(data)
        else:
            shutil.copy(os.path.join(ROOT, p), os.path.join(src, f))
    if rev:
        data = subprocess.run(["git", "show", f"{rev}:include/mg.h"], cwd=ROOT, check=True, capture_output=True).stdout
        open(os.path.join(inc, "mg.h"), "wb").write(data)
    else:
        shutil.copy(os.path.join(ROOT, "include", "mg.h"), os.path.join(inc, "mg.h"))
    flags = [f for f in B.FLAGS if not f.startswith("-I")] + ["-I" + inc] + os.environ.get("MG_AB_DEFS", "").split()
    objs = []
    procs = []
    for s in B.SOURCES:
        o = os.path.join(out, s + ".o")
        procs.append(subprocess.Popen([B.NVCC] + flags + ["-c", os.path.join(src, s), "-o", o]))
        objs.append(o)
    for p in procs:
        if p.wait() != 0:
            raise SystemExit("compile failed")
    subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", os.path.join(out, "libmg.so")]
                   + objs + ["-lcufft", "-lcublas"], check=True)
    for o in objs:
        os.remove(o)
    print(os.path.join(out, "libmg.so"))


if __name__ == "__main__":
    main()
