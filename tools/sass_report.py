"""SASS evidence for the blend kernels (north star: "absence of SFU ops in blend",
FP32 pipe): per k_blend16 instantiation the opcode histogram of the whole
kernel and of its hottest loop (the candidate walk), and the count of MUFU /
FFMA2 / FMUL2 / FADD2 instructions; then the walk loop's listing for the
headline poly-1 kernel.

    python tools/sass_report.py [paper_2603_18707_b200/_build/blend.o] > profiles/rNN_sass_blend16.txt
"""
import collections
import re
import subprocess
import sys

OBJ = sys.argv[1] if len(sys.argv) > 1 else "paper_2603_18707_b200/_build/blend.o"
sass = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)[1:]
INSN = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)")


def demangle(name):
    m = re.search(r"k_blend16ILi(\d)ELi(\d)ELi(\d)ELb(\d)E", name)
    if not m:
        return None
    kind, order, mode, count = m.groups()
    kname = "exp" if kind == "0" else f"poly{order}"
    return f"k_blend16<{kname}, {'quadric' if mode == '0' else 'alpha'}-threshold, count={count}>"


def parse(body):
    out = []
    for line in body.splitlines():
        m = INSN.search(line)
        if m:
            out.append((int(m.group(1), 16), m.group(3), line.strip()))
    return out


def walk_loop(ins):
    """The innermost backward branch that contains FFMA2s: the candidate walk."""
    best = None
    for addr, op, line in ins:
        m = re.search(r"BRA\s+(?:`\(.*?\)\s*)?0x([0-9a-f]+)", line)
        if op.startswith("BRA") and m:
            tgt = int(m.group(1), 16)
            if tgt < addr:
                body = [x for x in ins if tgt <= x[0] <= addr]
                n2 = sum(1 for x in body if x[1].startswith(("FFMA2", "FMUL2", "FADD2")))
                if n2 and (best is None or len(body) < len(best)):
                    best = body
    return best or []


print(__doc__.split("\n\n")[0])
print(f"\nobject: {OBJ}\n")
headline = None
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    label = demangle(name)
    if not label:
        continue
    ins = parse(f)
    ops = collections.Counter(op.split(".")[0] for _, op, _ in ins)
    loop = walk_loop(ins)
    lops = collections.Counter(op.split(".")[0] for _, op, _ in loop)
    mufu = [op for _, op, _ in ins if op.startswith("MUFU")]
    print(f"== {label}")
    print(f"   instructions {len(ins)}; MUFU total {len(mufu)} {dict(collections.Counter(mufu))}")
    print(f"   walk loop: {len(loop)} instructions; MUFU in loop {lops.get('MUFU', 0)}; "
          f"FFMA2/FMUL2/FADD2 {lops.get('FFMA2', 0)}/{lops.get('FMUL2', 0)}/{lops.get('FADD2', 0)}; "
          f"FFMA/FMUL/FADD {lops.get('FFMA', 0)}/{lops.get('FMUL', 0)}/{lops.get('FADD', 0)}; "
          f"LDS {lops.get('LDS', 0)}; FSETP {lops.get('FSETP', 0)}; FSEL {lops.get('FSEL', 0)}; "
          f"FMNMX {lops.get('FMNMX', 0)}")
    if "poly1, quadric-threshold, count=0" in label:
        headline = loop
if headline:
    print("\n== walk loop of k_blend16<poly1, quadric-threshold, count=0> (headline kernel)")
    for _, _, line in headline:
        print("   " + re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", line))
