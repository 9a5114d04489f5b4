"""Instruction mix of a SASS region: python tools/sass_mix.py <lib.so> <function-substring> [start_line end_line]
Counts opcodes (with FMA-pipe / ALU-pipe classification) in the given instruction-index range,
or in the whole function."""
import re
import subprocess
import sys
from collections import Counter

lib, fun = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", txt)
body = next(b for b in blocks[1:] if fun in b.split("\n", 1)[0])
ins = [l for l in body.split("\n") if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
ops = []
for l in ins:
    s = l.split("*/", 1)[1].strip()
    s = re.sub(r"^@!?U?P\w+\s+", "", s)
    ops.append(s.split()[0].rstrip(";"))
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, len(ops))
c = Counter(ops[lo:hi])
fma = sum(v * (2 if k.startswith("IMAD.WIDE") or k.startswith("IMAD.HI") else 1)
          for k, v in c.items() if k.startswith("IMAD"))
alu = sum(v for k, v in c.items() if k.split(".")[0] in ("IADD3", "LOP3", "SHF", "SEL", "ISETP", "MOV", "LEA", "PRMT", "VIADD", "IABS", "FLO", "POPC"))
for k, v in c.most_common():
    print(f"{v:5d} {k}")
print(f"total={hi-lo} fma_slots(WIDE/HI=2)={fma} alu~={alu}")
