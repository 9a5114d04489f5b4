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
mis = [i for i, (_, s) in enumerate(ins) if marker in s]
# innermost backward branch whose loop body contains a marker instruction
best = None
for i, (a, s) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?(?:`\()?.*?0x([0-9a-f]+)", s)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt not in addr_idx or addr_idx[tgt] >= i:
        continue
    lo_i = addr_idx[tgt]
    nmark = sum(1 for mi in mis if lo_i <= mi <= i)
    if nmark and (best is None or (i - lo_i) < (best[1] - best[0])):
        best = (lo_i, i, nmark)
lo, hi, nmark = best
ops = []
for _, s in ins[lo:hi + 1]:
    s = re.sub(r"^@!?U?P\w+\s+", "", s)
    ops.append(s.split()[0])
c = Counter(ops)
fma = sum(v * (2 if (k.startswith("IMAD.WIDE") or k.startswith("IMAD.HI")) else 1) for k, v in c.items() if k.startswith("IMAD"))
alu = sum(v for k, v in c.items() if k.split(".")[0] in ("IADD3", "LOP3", "SHF", "SEL", "ISETP", "MOV", "LEA", "PRMT", "VIADD", "POPC", "FLO", "I2FP"))
for k, v in c.most_common():
    print(f"{v:5d} {k}")
print(f"loop [{lo},{hi}] instructions={hi-lo+1} markers={nmark} fma_slots(WIDE/HI=2)={fma} alu~={alu}")
