"""Builds an alternative library _ab/<name>.so with extra nvcc defines on some
sources (A/B timing experiments; the product build is untouched):

    python tools/ab_variant.py NAME [-DFOO=1 ...] [--src blend.cu,...]

Objects of the other sources are reused from the product build
(paper_2603_18707_b200/_build). Run the variants with tools/ab.sh or
PS_B200_LIB=_ab/NAME.so.
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_18707_b200 import build as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("defines", nargs="*")
ap.add_argument("--src", default="blend.cu")
ap.add_argument("--from", dest="from_dir", default=None, help="take the --src files from this directory")
a, unknown = ap.parse_known_args()
a.defines += unknown
B.build()
out = os.path.join(ROOT, "_ab")
os.makedirs(out, exist_ok=True)
srcs = a.src.split(",")
objs = []
for src, extra in B.SOURCES:
    obj = os.path.join(B.BUILD, os.path.splitext(src)[0] + ".o")
    if src in srcs:
        obj = os.path.join(out, f"{a.name}_{os.path.splitext(src)[0]}.o")
        cmd = B._cmd(src, extra + list(a.defines), obj)
        if a.from_dir:
            cmd[cmd.index(os.path.join(B.CSRC, src))] = os.path.join(a.from_dir, src)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stdout + r.stderr)
        with open(obj + ".ptxas.txt", "w") as fh:
            fh.write(r.stderr)
    objs.append(obj)
lib = os.path.join(out, f"{a.name}.so")
link = [B._nvcc(), "-ccbin", B._host_cxx(), "-shared", *B.ARCH, "-o", lib, *objs, "-cudart", "static",
        "-Xlinker", f"--version-script={os.path.join(B.CSRC, 'exports.map')}"]
r = subprocess.run(link, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
print(lib)
