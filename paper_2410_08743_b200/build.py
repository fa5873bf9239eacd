"""Builds libgsb200.so in-tree with nvcc for sm_100a (no JIT cache, no torch).

Each translation unit compiles in parallel to build/*.o, then one nvcc link
produces paper_2410_08743_b200/libgsb200.so (git-ignored, travels with the
gpurun snapshot).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
OUT = os.path.join(PKG, "libgsb200.so")
OBJ = os.path.join(PKG, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr"]
FLAGS += os.environ.get("GSB_NVCC_EXTRA", "").split()  # experiment knobs (e.g. -DGSB_BWD_MIN_BLOCKS=8)


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cpp")))


def _headers():
    return glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "gsb200.h")]


def source_hash() -> str:
    """SHA-256 over every source, header and compiler flag of the library; the
    build stamps it into the .so (gsb_build_id) and beside it (OUT + '.id'), so
    a shipped binary is reused only when it was built from exactly these sources."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted(sources() + _headers()):
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def needs_build() -> bool:
    if not os.path.exists(OUT) or not os.path.exists(OUT + ".id"):
        return True
    with open(OUT + ".id") as fh:
        return fh.read().strip() != source_hash()


def _obj(src):
    return os.path.join(OBJ, os.path.basename(src) + ".o")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max(os.path.getmtime(h) for h in _headers())

    def compile_one(src):
        o = _obj(src)
        if not force and os.path.exists(o) and os.path.getmtime(o) > max(os.path.getmtime(src), hdr_t):
            return o
        cmd = [NVCC] + FLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-c", src, "-o", o]
        r = subprocess.run(cmd, cwd=PKG, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return o

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    sh = source_hash()
    id_src = os.path.join(OBJ, "build_id.cpp")
    with open(id_src, "w") as fh:
        fh.write(f'extern "C" const char* gsb_build_id(void) {{ return "{sh}"; }}\n')
    id_obj = id_src + ".o"
    subprocess.check_call(["g++", "-O2", "-fPIC", "-c", id_src, "-o", id_obj])
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", OUT + ".tmp"] + objs + [id_obj], cwd=PKG)
    os.replace(OUT + ".tmp", OUT)
    with open(OUT + ".id", "w") as fh:
        fh.write(sh + "\n")
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
