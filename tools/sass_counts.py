"""SASS instruction mix per output sample of each hot loop in libsquares.so (SURVEY.md 7 step 8:
"SASS instructions per output").  CPU-only (cuobjdump).  Writes profiles/<tag>_sass_counts.json.

    python tools/sass_counts.py r01
Pipe classes: FMA-heavy = IMAD* (WIDE/HI counted as 2 slots), ALU = integer add/logic/shift/
select/move forms, LSU = shared/global memory ops.
"""
import json
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2004_06278_b200", "libsquares.so")
ALU = ("IADD3", "LOP3", "SHF", "SEL", "ISETP", "MOV", "LEA", "PRMT", "VIADD", "IABS", "POPC", "FLO", "I2FP", "IMNMX", "VIMNMX")

# kernel symbol substring, loop marker, samples per loop iteration, description
LOOPS = [
    ("fill_kernelILi0ELb1ELb0E", "STG.E.ENL2.256", 16, "c2 u32 fill (key by value), per lane-chunk of 16"),
    ("fill_kernelILi1ELb1ELb0E", "STG.E.ENL2.256", 8, "c3 u64 fill (key by value), per lane-chunk of 8"),
    ("fill_kernelILi2ELb0ELb0E", "STG.E.ENL2.256", 16, "c4 f32 fill (device keys), per lane-chunk of 16"),
]


def functions(txt):
    for blk in re.split(r"\n\s*Function : ", txt)[1:]:
        name = blk.split("\n", 1)[0].strip()
        ins = []
        for line in blk.split("\n"):
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        yield name, ins


def opcode(s):
    return re.sub(r"^@!?U?P\w+\s+", "", s).split()[0]


def innermost_loop(ins, marker):
    idx = {a: i for i, (a, _) in enumerate(ins)}
    best = None
    for i, (_, s) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?(?:`\()?.*?0x([0-9a-f]+)", s)
        if not m:
            continue
        t = int(m.group(1), 16)
        if t in idx and idx[t] < i and any(marker in x for _, x in ins[idx[t]:i + 1]):
            if best is None or i - idx[t] < best[1] - best[0]:
                best = (idx[t], i)
    return best


def classify(c, samples):
    fma = sum(v * (2 if k.startswith(("IMAD.WIDE", "IMAD.HI")) else 1) for k, v in c.items() if k.startswith("IMAD"))
    alu = sum(v for k, v in c.items() if k.split(".")[0] in ALU)
    lsu = sum(v for k, v in c.items() if k.split(".")[0] in ("ATOMS", "STG", "LDS", "STS", "LDG", "RED"))
    mul = sum(v for k, v in c.items() if k in ("IMAD", "IMAD.WIDE.U32", "IMAD.HI.U32"))
    tot = sum(c.values())
    return {"instructions_per_sample": tot / samples, "fma_slots_per_sample": fma / samples,
            "multiply_instructions_per_sample": mul / samples, "alu_per_sample": alu / samples,
            "lsu_per_sample": lsu / samples, "mix": dict(c.most_common())}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    fns = dict(functions(txt))
    out = {"lib": os.path.relpath(LIB, ROOT), "method": "innermost loop containing the marker; "
           "WIDE/HI = 2 FMA-heavy slots", "kernels": {}}
    for sub, marker, samples, desc in LOOPS:
        name, ins = next((n, i) for n, i in fns.items() if sub in n)
        lo, hi = innermost_loop(ins, marker)
        c = Counter(opcode(s) for _, s in ins[lo:hi + 1])
        out["kernels"][desc] = {"symbol": name, **classify(c, samples)}
    # fused: the unmasked epoch block (32 samples) = the straight-line code between the first two
    # branches after the epoch-loop head that contains 32 ATOMS
    name, ins = next((n, i) for n, i in fns.items() if "fused_kernelILb0ELb0E" in n)
    br = [i for i, (_, s) in enumerate(ins) if opcode(s).startswith("BRA")]
    for a, b in zip(br, br[1:]):
        c = Counter(opcode(s) for _, s in ins[a + 1:b])
        if c.get("ATOMS.ADD", 0) == 32:
            out["kernels"]["c5 fused statistics, per 32-sample epoch block"] = {"symbol": name, **classify(c, 32)}
            break
    path = os.path.join(ROOT, "profiles", f"{tag}_sass_counts.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    for k, v in out["kernels"].items():
        print(f"{k}: {v['instructions_per_sample']:.2f} instr/sample, {v['fma_slots_per_sample']:.2f} FMA slots, "
              f"{v['alu_per_sample']:.2f} ALU, {v['multiply_instructions_per_sample']:.2f} multiplies")


if __name__ == "__main__":
    main()
