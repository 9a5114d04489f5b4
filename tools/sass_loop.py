"""Instruction mix of the innermost loop containing a given opcode (default STG.E.ENL2.256).
python tools/sass_loop.py <lib.so> <function-substring> [opcode]"""
import re
import subprocess
import sys
from collections import Counter

lib, fun = sys.argv[1], sys.argv[2]
marker = sys.argv[3] if len(sys.argv) > 3 else "STG.E.ENL2.256"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", txt)
body = next(b for b in blocks[1:] if fun in b.split("\n", 1)[0])
ins = []
for l in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
mi = next(i for i, (_, s) in enumerate(ins) if marker in s)
# innermost backward branch that jumps to <= marker and sits after it
best = None
for i, (a, s) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\()?.*?0x([0-9a-f]+)", s)
    if m and i > mi:
        tgt = int(m.group(1), 16)
        if tgt in addr_idx and addr_idx[tgt] <= mi:
            if best is None or (i - addr_idx[tgt]) < (best[1] - best[0]):
                best = (addr_idx[tgt], i)
lo, hi = best
ops = []
for _, s in ins[lo:hi + 1]:
    s = re.sub(r"^@!?U?P\w+\s+", "", s)
    ops.append(s.split()[0])
c = Counter(ops)
fma = sum(v * (2 if (k.startswith("IMAD.WIDE") or k.startswith("IMAD.HI")) else 1) for k, v in c.items() if k.startswith("IMAD"))
alu = sum(v for k, v in c.items() if k.split(".")[0] in ("IADD3", "LOP3", "SHF", "SEL", "ISETP", "MOV", "LEA", "PRMT", "VIADD", "POPC", "FLO", "I2FP"))
for k, v in c.most_common():
    print(f"{v:5d} {k}")
print(f"loop [{lo},{hi}] instructions={hi-lo+1} fma_slots(WIDE/HI=2)={fma} alu~={alu}")
