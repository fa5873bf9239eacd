"""Builds oracle/_ref from the reference's OWN sources — TEST INFRASTRUCTURE ONLY.

Compiles /root/reference/proj/src/*.cpp in place (read-only, never copied)
against the clean-room Eigen / doctest / libpng shim in oracle/shim, with the
reference's Release flags (-O3 -DNDEBUG, C++20; proj/CMakeLists.txt:3-10) and
no FMA contraction, into:

  oracle/_ref/libgsopt_ref.so   reference library + oracle/ref_capi.cpp (C ABI)
  oracle/_ref/test_*            the reference's own doctest suites
  oracle/_ref/acceptance        the reference's acceptance runner

nlohmann/json (scene_io.cpp, run_config.cpp) comes from the copy bundled with
cudnn_frontend in this image. The outputs are git-ignored but travel to the
GPU box with the gpurun snapshot; /root/reference is never read there (this
script is a no-op when it is absent).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("GSOPT_REF_ROOT", "/root/reference/proj")
OUT = os.path.join(HERE, "_ref")
OBJ = os.path.join(OUT, "obj")
SHIM = os.path.join(HERE, "shim")
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
CXX = os.environ.get("CXX", "g++")
FLAGS = ["-std=c++20", "-O3", "-DNDEBUG", "-ffp-contract=off", "-fPIC", "-pthread", "-w",
         "-I" + SHIM, "-I" + os.path.join(REF, "include"), "-I" + os.path.join(REF, "tests"), "-I" + JSON_DIR,
         "-I" + HERE]
LIB_SOURCES = ["core", "lie", "sh", "scene", "image", "rasterizer", "losses", "eval", "trainer", "pipelines",
               "ply", "scene_io", "synth", "run_config"]
TESTS = ["test_lie", "test_scene", "test_rasterizer", "test_losses", "test_eval", "test_trainer", "test_io",
         "test_config"]
LIB = os.path.join(OUT, "libgsopt_ref.so")


def available() -> bool:
    return os.path.isdir(os.path.join(REF, "src"))


def _deps():
    return glob.glob(os.path.join(SHIM, "*")) + glob.glob(os.path.join(SHIM, "Eigen", "*")) + [
        os.path.join(HERE, "ref_capi.cpp"), os.path.join(HERE, "gsopt_oracle.h"), os.path.abspath(__file__)]


def _stale(target, extra=()):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in list(_deps()) + list(extra))


def _compile(src, obj):
    if not _stale(obj, [src]):
        return obj
    r = subprocess.run([CXX] + FLAGS + ["-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"{src}:\n{r.stderr[-4000:]}")
    return obj


def build(force: bool = False) -> str | None:
    if not available():
        return LIB if os.path.exists(LIB) else None
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(f)
    jobs = [(os.path.join(REF, "src", s + ".cpp"), os.path.join(OBJ, s + ".o")) for s in LIB_SOURCES]
    jobs.append((os.path.join(HERE, "ref_capi.cpp"), os.path.join(OBJ, "ref_capi.o")))
    jobs += [(os.path.join(REF, "tests", t + ".cpp"), os.path.join(OBJ, t + ".o")) for t in
             TESTS + ["test_main", "acceptance"]]
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = dict(zip([j[1] for j in jobs], ex.map(lambda j: _compile(*j), jobs)))
    lib_objs = [os.path.join(OBJ, s + ".o") for s in LIB_SOURCES]
    if force or _stale(LIB, lib_objs + [os.path.join(OBJ, "ref_capi.o")]):
        subprocess.check_call([CXX, "-shared", "-pthread", "-o", LIB + ".tmp"] + lib_objs +
                              [os.path.join(OBJ, "ref_capi.o")])
        os.replace(LIB + ".tmp", LIB)
    archive = os.path.join(OBJ, "libgsopt.a")
    if force or _stale(archive, lib_objs):
        if os.path.exists(archive):
            os.remove(archive)
        subprocess.check_call(["ar", "rcs", archive] + lib_objs)

    def link(name, extra):
        exe = os.path.join(OUT, name)
        if force or _stale(exe, [os.path.join(OBJ, name + ".o"), archive]):
            subprocess.check_call([CXX, "-pthread", "-o", exe, os.path.join(OBJ, name + ".o")] + extra + [archive])
    with ThreadPoolExecutor(max_workers=8) as ex:
        list(ex.map(lambda t: link(t, [os.path.join(OBJ, "test_main.o")]), TESTS))
    link("acceptance", [])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
