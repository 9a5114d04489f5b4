"""Opcode mix of the innermost loop (largest-instruction-count loop containing `marker`) of each
function matching a substring: python exp/loopmix.py <binary> <func-substring> [marker]"""
import re, subprocess, sys
from collections import Counter
binp, fun = sys.argv[1], sys.argv[2]
marker = sys.argv[3] if len(sys.argv) > 3 else "IMAD"
txt = subprocess.run(["cuobjdump", "-sass", binp], capture_output=True, text=True).stdout
for blk in re.split(r"\n\s*Function : ", txt)[1:]:
    name = blk.split("\n", 1)[0].strip()
    if fun not in name:
        continue
    ins = []
    for l in blk.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
    idx = {a: i for i, (a, _) in enumerate(ins)}
    best = None
    for i, (a, s) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?(?:`\()?.*?0x([0-9a-f]+)", s)
        if not m: continue
        t = int(m.group(1), 16)
        if t in idx and idx[t] < i and any(marker in x for _, x in ins[idx[t]:i]):
            if best is None or i - idx[t] > best[1] - best[0]: best = (idx[t], i)
    if not best: continue
    ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", s).split()[0] for _, s in ins[best[0]:best[1] + 1])
    print(name, "loop", best, "n=", best[1] - best[0] + 1, dict(ops.most_common(12)))
