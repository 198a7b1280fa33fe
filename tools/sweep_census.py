"""Per-pair SASS census of the config-5 sweep kernels' main row loop (no-store form):
counts the instructions between the loop head (first LDS of the staged rows) and its
back-branch and divides by the pairs one iteration covers (2 rows x 16 columns)."""
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2402_00675_b200/libnttk_gpu.so"
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
NAMES = ["mont", "smont", "plantard", "mplantard"]
for f in funcs:
    m = re.match(r"\S*sweep_kernelILi(\d)ELi(\d+)ELb0E", f)
    if not m or m.group(2) == "0":
        continue
    ins = [re.sub(r"/\*[0-9a-f]{4}\*/\s+", "", l).strip().rstrip(" ;")
           for l in f.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
    ins = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", x).strip().rstrip(" ;") for x in ins]
    addr = [int(re.match(r"\s+/\*([0-9a-f]{4})\*/", l).group(1), 16)
            for l in f.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
    best = None
    for i, x in enumerate(ins):  # hottest backward branch = the row loop
        mm = re.match(r"BRA(?:\.U)? .*?(0x[0-9a-f]+)$", x)
        if mm and int(mm.group(1), 16) < addr[i]:
            j = addr.index(int(mm.group(1), 16))
            n_mul = sum(1 for y in ins[j:i + 1] if y.startswith("IMAD") and "MOV" not in y)
            if best is None or n_mul > best[0]:
                best = (n_mul, j, i)
    body = ins[best[1]:best[2] + 1]
    pairs = 16 * sum(1 for y in body if y.startswith("LDS"))
    ops = {}
    for x in body:
        op = x.split()[0] if not x.startswith("@") else x.split()[1]
        ops[op] = ops.get(op, 0) + 1
    fma = sum(v for k, v in ops.items() if k.startswith("IMAD") and not k.startswith("IMAD.MOV"))
    cyc = sum(v * (4 if k.startswith(("IMAD.HI", "IMAD.WIDE")) else 2)
              for k, v in ops.items() if k.startswith("IMAD") and not k.startswith("IMAD.MOV"))
    other = len(body) - fma
    print(f"{NAMES[int(m.group(1))]:9s} n{m.group(2)}: {len(body) / pairs:5.2f} instr/pair, "
          f"FMA-pipe {fma / pairs:4.2f} ({cyc / pairs:4.2f} cyc), other {other / pairs:4.2f}  "
          + " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda t: -t[1])[:8]))
