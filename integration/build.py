"""Builds the drop-in proof: the reference library (/root/reference/proj/src,
compiled in place, never copied) with integration/gsopt_b200.cpp — the
adapter over libgsb200's C ABI — linked INSTEAD OF src/rasterizer.cpp, and
the reference's own test drivers against it:

  integration/_build/acceptance_b200   tests/acceptance.cpp criteria (by number)
  integration/_build/test_<suite>_b200 the reference's doctest suites

The reference needs Eigen / doctest / libpng, which this image lacks; the
clean-room subsets in oracle/shim stand in (the same ones oracle/build_ref.py
uses, so the reference's own code is what runs). Outputs are git-ignored and
travel to the GPU box with the snapshot; /root/reference is only read here.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.environ.get("GSOPT_REF_ROOT", "/root/reference/proj")
OUT = os.path.join(HERE, "_build")
OBJ = os.path.join(OUT, "obj")
SHIM = os.path.join(ROOT, "oracle", "shim")
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
LIBDIR = os.path.join(ROOT, "paper_2410_08743_b200")
CXX = os.environ.get("CXX", "g++")
FLAGS = ["-std=c++20", "-O3", "-DNDEBUG", "-ffp-contract=off", "-fPIC", "-pthread", "-w",
         "-I" + SHIM, "-I" + os.path.join(REF, "include"), "-I" + os.path.join(REF, "tests"), "-I" + JSON_DIR,
         "-I" + os.path.join(ROOT, "include")]
# every reference library source except src/rasterizer.cpp (replaced by the adapter)
LIB_SOURCES = ["core", "lie", "sh", "scene", "image", "losses", "eval", "trainer", "pipelines", "ply", "scene_io",
               "synth", "run_config"]
SUITES = ["test_rasterizer", "test_trainer", "test_losses", "test_scene"]
LINK = ["-L" + LIBDIR, "-lgsb200", "-Wl,-rpath,$ORIGIN/../../paper_2410_08743_b200", "-pthread"]


def available() -> bool:
    return os.path.isdir(os.path.join(REF, "src"))


def _compile(src, obj):
    deps = [src, os.path.abspath(__file__), os.path.join(ROOT, "include", "gsb200.h")] + glob.glob(
        os.path.join(SHIM, "*")) + glob.glob(os.path.join(SHIM, "Eigen", "*"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    r = subprocess.run([CXX] + FLAGS + ["-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"{src}:\n{r.stderr[-4000:]}")
    return obj


def build() -> str | None:
    if not available():
        return OUT if os.path.exists(os.path.join(OUT, "acceptance_b200")) else None
    os.makedirs(OBJ, exist_ok=True)
    jobs = [(os.path.join(REF, "src", s + ".cpp"), os.path.join(OBJ, s + ".o")) for s in LIB_SOURCES]
    jobs.append((os.path.join(HERE, "gsopt_b200.cpp"), os.path.join(OBJ, "gsopt_b200.o")))
    jobs.append((os.path.join(HERE, "acceptance_b200.cpp"), os.path.join(OBJ, "acceptance_b200.o")))
    jobs += [(os.path.join(REF, "tests", t + ".cpp"), os.path.join(OBJ, t + ".o")) for t in SUITES + ["test_main"]]
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda j: _compile(*j), jobs))
    lib_objs = [os.path.join(OBJ, s + ".o") for s in LIB_SOURCES] + [os.path.join(OBJ, "gsopt_b200.o")]

    def link(name, objs):
        exe = os.path.join(OUT, name)
        subprocess.check_call([CXX, "-o", exe] + objs + lib_objs + LINK)
        return exe

    link("acceptance_b200", [os.path.join(OBJ, "acceptance_b200.o")])
    for t in SUITES:
        link(t + "_b200", [os.path.join(OBJ, t + ".o"), os.path.join(OBJ, "test_main.o")])
    return OUT


if __name__ == "__main__":
    print(build())
