"""Builds the native library paper_2603_18707_b200/libpolysplat_b200.so in-tree.

nvcc cross-compiles for sm_100a only (`-gencode arch=compute_100a,code=sm_100a`);
no GPU is needed to build. The fp64-exact stages (exact_kernels.cu) are compiled
with `-fmad=false` and all host code with `-ffp-contract=off`, which is what makes
the preprocess bit-identical to the reference's FMA-free build.

    python -m paper_2603_18707_b200.build [--force] [-j N]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libpolysplat_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _host_cxx() -> str:
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


# (source, extra nvcc flags)
SOURCES = [
    ("exact_kernels.cu", ["-fmad=false"]),
    ("blend.cu", []),
    ("sort.cu", []),
    ("binning.cu", []),
    ("utils.cu", []),
    ("metrics.cu", []),
    ("context.cu", []),
    ("hostmath.cpp", []),
    ("synth.cpp", []),
    ("ply.cpp", []),
]
HEADERS = ["common.cuh", "exact_math.cuh", "kernels.h", "tile_sort.cuh"]


def _cmd(src: str, extra: list[str], obj: str) -> list[str]:
    nvcc = _nvcc()
    base = [nvcc, "-ccbin", _host_cxx(), "-std=c++17", "-O3", "-lineinfo", *ARCH,
            "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-Xptxas", "-v",
            f"-I{INCLUDE}", f"-I{CSRC}"]
    if src.endswith(".cpp"):
        base += ["-x", "c++"]
    return base + extra + ["-c", os.path.join(CSRC, src), "-o", obj]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(CSRC, "exports.map"),
        os.path.join(INCLUDE, "polysplat_b200.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, jobs: int = 8, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs, todo = [], []
    for src, extra in SOURCES:
        obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            todo.append((src, extra, obj))

    def run(item):
        src, extra, obj = item
        r = subprocess.run(_cmd(src, extra, obj), capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        with open(obj + ".ptxas.txt", "w") as fh:
            fh.write(r.stderr)
        return src

    if todo:
        with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
            for src in ex.map(run, todo):
                if verbose:
                    print(f"  compiled {src}", file=sys.stderr)
    if todo or not os.path.exists(LIB):
        link = [_nvcc(), "-ccbin", _host_cxx(), "-shared", *ARCH, "-o", LIB, *objs, "-cudart", "static",
                "-Xlinker", f"--version-script={os.path.join(CSRC, 'exports.map')}"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.j, verbose=True))


if __name__ == "__main__":
    main()
