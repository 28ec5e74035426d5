"""Builds the native library in-tree: paper_2404_12063_b200/_lib/libvpinn_b200.so.

CUDA sources (csrc/gpu/*.cu) are compiled for sm_100a only
(-gencode arch=compute_100a,code=sm_100a -lineinfo), host C++ (csrc/host/*.cpp)
with g++; translation units build in parallel and are skipped when newer than
every header they could include.  Run: python -m paper_2404_12063_b200.build_native
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "libvpinn_b200.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX_HOST", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"
INCLUDES = ["-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CSRC, "gpu"),
            "-I" + os.path.join(CSRC, "host")]
if os.path.isdir(os.path.join(JSON_INC, "nlohmann")):
    INCLUDES.append("-I" + JSON_INC)


def _headers():
    hs = []
    for pat in ("gpu/*.cuh", "gpu/*.h", "host/*.hpp", "host/*.h"):
        hs += glob.glob(os.path.join(CSRC, pat))
    hs += glob.glob(os.path.join(ROOT, "include", "*.h"))
    return hs


def _stale(src, obj, hdr_mtime):
    if not os.path.exists(obj):
        return True
    m = os.path.getmtime(obj)
    return os.path.getmtime(src) > m or hdr_mtime > m


def _compile(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    return cmd, r.returncode, r.stdout + r.stderr


def build(verbose: bool = False, jobs: int | None = None, force: bool = False) -> str:
    # diagnostics builds (e.g. VPINN_EXTRA_NVCC=-DVPG_PHASE_CLOCK=1) rebuild everything
    extra = os.environ.get("VPINN_EXTRA_NVCC", "").split()
    force = force or bool(extra)
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    hdr_mtime = max([os.path.getmtime(h) for h in _headers()] + [0.0])
    cu = sorted(glob.glob(os.path.join(CSRC, "gpu", "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    objs, cmds = [], []
    for s in cu:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(s, o, hdr_mtime):
            # assemble.cu: no FMA contraction, so the double geometry is the
            # host's bits (the host is built with -ffp-contract=off)
            per_file = ["--fmad=false"] if os.path.basename(s) == "assemble.cu" else []
            cmds.append([NVCC, "-std=c++20", *ARCH, "-O3", "-lineinfo", "-Xptxas", "-v", *extra, *per_file,
                         "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
                         "--expt-relaxed-constexpr", *INCLUDES, "-c", s, "-o", o])
    for s in cpp:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(s, o, hdr_mtime):
            cmds.append([CXX, "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall",
                         "-Wno-unused-parameter", *INCLUDES, "-I/usr/local/cuda/include",
                         "-c", s, "-o", o])
    if cmds:
        with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
            for cmd, rc, out in ex.map(_compile, cmds):
                if verbose or rc != 0:
                    sys.stderr.write(" ".join(cmd[-3:]) + "\n" + out)
                if rc != 0:
                    raise RuntimeError(f"native build failed: {cmd[-3]}")
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        link = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ldl", "-lpthread"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="--force" in sys.argv))
