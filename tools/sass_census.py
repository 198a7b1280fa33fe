#!/usr/bin/env python3
"""SASS census of the engine's kernels (cuobjdump -sass of libnttk_gpu.so).

For every kernel it finds the hottest loop (the backward-branch region with the most
IMAD-family instructions), counts opcodes there, and derives per-butterfly costs:
one loop iteration of a fast256 consumer warp transforms 2 polynomials, i.e. 64
butterflies per thread (8 layers x 8) or 56 (7 layers).  The fmaheavy estimate uses the
measured issue costs (profiles/r1a_imad_microbench.txt): IMAD 2 cycles, IMAD.HI /
IMAD.WIDE 4 cycles per warp instruction on one SM sub-partition.
Usage: python tools/sass_census.py [lib.so] [name-regex] [--ops] [--json OUT]
  --ops: opcode breakdown; --json OUT: also write the rows (+ the library's sha256) for
  bench.py's executed-instruction IMAD roof
"""
import re
import subprocess
import sys
from collections import Counter

OPS = "--ops" in sys.argv
sys.argv = [a for a in sys.argv if a != "--ops"]
JSON = None
if "--json" in sys.argv:
    i = sys.argv.index("--json")
    JSON = sys.argv[i + 1]
    del sys.argv[i:i + 2]
rows = []

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2402_00675_b200/libnttk_gpu.so"
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else
                 r"tma_kernel.*(ImprovedN16ILb0EEEtLi8|ImprovedN32EjLi8|HarveyILi16ELb0EEEtLi8|HarveyILi32ELb0EEEjLi8|SmontILi16EEtLi8|SmontILi32EEjLi8)"
                 r"|polymul256_tma_kernel.*(ImprovedN16ILb0EEEtLi7|HarveyLazy16EtLi7|SmontLazy16EtLi7)")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
FMA2 = ("IMAD", "IMAD.IADD", "IMAD.MOV", "IMAD.MOV.U32", "IMAD.SHL.U32", "IMAD.X", "IMAD.U32")
FMA4 = ("IMAD.HI.U32", "IMAD.WIDE.U32", "IMAD.WIDE", "IMAD.HI")
print(f"{'kernel':70s} {'instr':>5s} {'IMAD':>5s} {'.HI':>4s} {'.WIDE':>5s} {'IADD':>5s} "
      f"{'alu':>4s} {'lsu':>4s} {'fmaheavy_cyc':>12s} {'per_bfly':>8s}")
for part in re.split(r"\n\s+Function : ", txt)[1:]:
    name = part.split("\n", 1)[0]
    if not pat.search(name):
        continue
    ins = []
    for line in part.split("\n"):
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(?:\.[A-Z0-9_]+)*)([^;]*);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    best, best_n = None, -1
    for a, op, rest in ins:
        t = re.search(r"0x([0-9a-f]+)", rest)
        if op.startswith("BRA") and t and int(t.group(1), 16) < a:
            lo = int(t.group(1), 16)
            if any(lo <= x <= a and o == "EXIT" for x, o, _ in ins):
                continue  # a retry stub branching back over the producer / kernel exits
            n = sum(1 for x, o, _ in ins if lo <= x <= a and o.startswith("IMAD"))
            # the most IMADs; among equal counts the tightest region (the retry stubs of
            # mbarrier waits branch back from the end of the kernel over everything)
            if n > best_n or (n == best_n and a - lo < best[1] - best[0]):
                best, best_n = (lo, a), n
    if not best:
        continue
    c = Counter(o for x, o, _ in ins if best[0] <= x <= best[1])
    n = sum(c.values())
    imad = sum(v for k, v in c.items() if k in FMA2 or (k.startswith("IMAD") and k not in FMA4))
    hi = c.get("IMAD.HI.U32", 0) + c.get("IMAD.HI", 0)
    wide = c.get("IMAD.WIDE.U32", 0) + c.get("IMAD.WIDE", 0)
    iadd = sum(v for k, v in c.items() if k.startswith("IADD3"))
    alu = sum(v for k, v in c.items() if k.startswith(("IADD3", "LOP3", "SHF", "LEA", "VIMNMX", "IMNMX", "ISETP", "SEL", "PRMT")))
    lsu = sum(v for k, v in c.items() if k.startswith(("LDS", "STS", "LDG", "STG", "SYNCS")))
    fcyc = 2 * imad + 4 * (hi + wide)
    bfly = 56 if "Li7E" in name else 64
    short = re.sub(r"_ZN9nttk_b200\w*?_GLOBAL__N__\w+?\d+(fwd|inv)", r"\1", name)[:70]
    print(f"{short:70s} {n:5d} {imad:5d} {hi:4d} {wide:5d} {iadd:5d} {alu:4d} {lsu:4d} "
          f"{fcyc:12d} {fcyc / bfly:8.2f}")
    rows.append({"kernel": name, "instr": n, "imad": imad, "imad_hi": hi, "imad_wide": wide,
                 "iadd3": iadd, "alu": alu, "lsu": lsu, "fmaheavy_cycles_per_iter": fcyc,
                 "polys_per_iter": 2, "ops": dict(c.most_common())})
    if OPS:
        print("    " + "  ".join(f"{k}:{v}" for k, v in c.most_common()))

if JSON:
    import hashlib
    import json

    import os

    with open(lib, "rb") as fh:
        sha = hashlib.sha256(fh.read()).hexdigest()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from bench import kernel_source_sha

    with open(JSON, "w") as fh:
        json.dump({"lib": lib, "lib_sha256": sha, "src_sha256": kernel_source_sha(),
                   "note": "hottest consumer loop per kernel; one iteration = 2 polynomials per "
                           "warp; fmaheavy cycles = 2 x IMAD + 4 x (IMAD.HI + IMAD.WIDE) per "
                           "warp on one SM sub-partition", "rows": rows}, fh, indent=1)
