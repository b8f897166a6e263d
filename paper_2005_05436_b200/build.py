"""In-tree build of the sm_100a library (nvcc) — no JIT cache, no pip install.

    python -m paper_2005_05436_b200.build        # builds _build/libtopo_b200.so

The shared library is what travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_build")
LIB = os.path.join(OUT_DIR, "libtopo_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-fopenmp", "-Xcompiler", "-Wall"]
SOURCES = ["capi.cu", "host_setup.cpp"]
HEADERS = ["kernels.cuh", "common.cuh", "control.h", "comm.h", "mg.cuh"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (CUDA 12.9 toolkit required)")


def _stale() -> bool:
    return _stale_lib(LIB)


# the checked variant (device bounds asserts, TOPO_CHECK in common.cuh):
# tests/test_gpu_checked.py runs parity cases against it
LIB_CHECKED = os.path.join(OUT_DIR, "libtopo_b200_checked.so")


def _stale_lib(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "topo_capi.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Compile the library (and with checked=True also the checked variant);
    the translation units compile in parallel. Returns the library path."""
    variants = [(LIB, [])]
    if checked:
        variants.append((LIB_CHECKED, ["-DTOPO_CHECKED"]))
    variants = [(lib, fl) for lib, fl in variants if force or _stale_lib(lib)]
    if not variants:
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    nvcc = _nvcc()
    env = dict(os.environ)
    env.pop("CC", None)   # use the system host compiler (nvcc's default)
    env.pop("CXX", None)
    jobs, links = [], []
    for lib, extra in variants:
        tag = "" if not extra else "_checked"
        objs = []
        for src in SOURCES:
            obj = os.path.join(OUT_DIR, os.path.splitext(src)[0] + tag + ".o")
            cmd = [nvcc] + NVCC_FLAGS + extra + ["-c", os.path.join(CSRC, src), "-o", obj]
            if src.endswith(".cu") and verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)
            objs.append(obj)
        links.append((lib, objs))
    procs = [(cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                    text=True, env=env)) for cmd in jobs]
    for cmd, p in procs:
        out, err = p.communicate()
        _check(cmd, p.returncode, out, err)
    for lib, objs in links:
        tmp = lib + ".tmp"
        _run([nvcc] + ARCH + ["-shared", "-o", tmp] + objs + ["-lgomp", "-ldl"], env)
        os.replace(tmp, lib)
    return LIB


def _check(cmd, rc, out, err):
    if rc != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + out + err)
    if err.strip() and os.environ.get("TOPO_BUILD_VERBOSE"):
        sys.stderr.write(err)


def _run(cmd, env):
    r = subprocess.run(cmd, capture_output=True, text=True, env=env)
    _check(cmd, r.returncode, r.stdout, r.stderr)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                checked="--checked" in sys.argv))
