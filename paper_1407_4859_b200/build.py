"""Build libadha.so in-tree: nvcc for sm_100a, static cudart, -lineinfo.

    python paper_1407_4859_b200/build.py [--force] [-v]

(Run as a script: importing the package first would need the library it builds.)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libadha.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
          "-I", os.path.join(ROOT, "include")]


def sources():
    out = []
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cu", ".cpp")):
            out.append(os.path.join(CSRC, name))
    return out


def _deps():
    files = sources() + [os.path.join(CSRC, n) for n in os.listdir(CSRC) if n.endswith((".h", ".cuh"))]
    files.append(os.path.join(ROOT, "include", "adha.h"))
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB) -> str:
    """Compile every csrc/ source for sm_100a and link `lib`.  `defines` (e.g. ADHA_PHASE_TIMING
    for the instrumented diagnostic library) go to every compile; such variants are linked to
    their own file under _build/, never to the product libadha.so."""
    if not force and not defines and up_to_date():
        return lib
    tag = "_".join(d.lower() for d in defines)
    bdir = os.path.join(BUILD, tag) if tag else BUILD
    os.makedirs(bdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [NVCC] + ARCH + COMMON + [f"-D{d}" for d in defines] + ["-c", src, "-o", obj]
        if src.endswith(".cu") and verbose:
            cmd += ["-Xptxas", "-v"]
        objs.append(obj)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode != 0:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    tmp = lib + ".tmp"
    link = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + ["-lpthread", "-lrt", "-ldl"]
    subprocess.check_call(link)
    os.replace(tmp, lib)
    return lib


def build_phase_timing() -> str:
    """The diagnostic library with per-phase clock64() counters in the tiled kernel
    (tools/phase_probe.py); not used by the package, the tests or the bench."""
    return build(force=True, defines=("ADHA_PHASE_TIMING",), lib=os.path.join(BUILD, "libadha_phase.so"))


if __name__ == "__main__":
    if "--phase-timing" in sys.argv:
        print(build_phase_timing())
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
