"""SASS instruction mix per output sample of each hot loop in libsquares.so (SURVEY.md 7 step 8:
"SASS instructions per output").  CPU-only (cuobjdump).  Writes profiles/<tag>_sass_counts.json.

    python tools/sass_counts.py r01
Pipe classes: FMA-heavy = IMAD* and VIADD (WIDE/HI counted as 2 slots), ALU = integer
add/logic/shift/select/move forms, LSU = shared/global memory ops.
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
    ("fill_kernelILi1ELb1ELb0E", "STG.E.ENL2.256", 16, "c3 u64 fill (key by value), per 2 lane-chunks of 8 (loop unrolled by 2)"),
    ("fill_kernelILi2ELb0ELb0E", "STG.E.ENL2.256", 16, "c4 f32 fill (device keys), per lane-chunk of 16"),
    ("fill_kernelILi0ELb0ELb0E", "STG.E.ENL2.256", 16, "c2 u32 fill (device keys), per lane-chunk of 16"),
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
    # VIADD issues to the FMA-heavy pipe on sm_100 (ncu smsp__inst_executed_pipe_fmaheavy counts
    # it: profiles/r02_c5_pipes.json), so it is counted there, not as ALU
    fma = sum(v * (2 if k.startswith(("IMAD.WIDE", "IMAD.HI")) else 1) for k, v in c.items()
              if k.startswith(("IMAD", "VIADD")))
    alu = sum(v for k, v in c.items() if k.split(".")[0] in ALU and not k.startswith("VIADD"))
    lsu = sum(v for k, v in c.items() if k.split(".")[0] in ("ATOMS", "STG", "LDS", "STS", "LDG", "RED"))
    mul = sum(v for k, v in c.items() if k in ("IMAD", "IMAD.WIDE.U32", "IMAD.HI.U32"))
    tot = sum(c.values())
    c = Counter({k: round(v, 3) for k, v in c.items()})
    return {"instructions_per_sample": tot / samples, "fma_slots_per_sample": fma / samples,
            "multiply_instructions_per_sample": mul / samples, "alu_per_sample": alu / samples,
            "lsu_per_sample": lsu / samples, "mix": dict(c.most_common())}


KEY_OF = {"c2 u32 fill (key by value), per lane-chunk of 16": "c2",
          "c3 u64 fill (key by value), per 2 lane-chunks of 8 (loop unrolled by 2)": "c3",
          "c4 f32 fill (device keys), per lane-chunk of 16": "c4",
          "c2 u32 fill (device keys), per lane-chunk of 16": "c2_devkeys",
          "c5 fused statistics (warp-specialised), generator tree + reducer slot, per 32 samples": "c5",
          "c5 fused statistics (lock-step kernel), per 32-sample epoch block": "c5_lockstep"}


def counts(lib: str = LIB) -> dict:
    """{description: {symbol, instructions_per_sample, fma_slots_per_sample, ...}} of the hot
    loops in `lib` (cuobjdump -sass; no GPU needed)."""
    txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    fns = dict(functions(txt))
    out = {}
    for sub, marker, samples, desc in LOOPS:
        name, ins = next((n, i) for n, i in fns.items() if sub in n)
        lo, hi = innermost_loop(ins, marker)
        c = Counter(opcode(s) for _, s in ins[lo:hi + 1])
        out[desc] = {"symbol": name, **classify(c, samples)}
    # fused, lock-step kernel (fused_kernel, SQ_FUSED_IMPL=0 builds): the unmasked epoch block
    # (32 samples) = the straight-line code between two branches that contains 32 ATOMS
    lock = [(n, i) for n, i in fns.items() if "12fused_kernelILb0ELb0E" in n]
    for name, ins in lock:
        br = [i for i, (_, s) in enumerate(ins) if opcode(s).startswith("BRA")]
        for a, b in zip(br, br[1:]):
            c = Counter(opcode(s) for _, s in ins[a + 1:b])
            if c.get("ATOMS.ADD", 0) == 32:
                out["c5 fused statistics (lock-step kernel), per 32-sample epoch block"] = {
                    "symbol": name, **classify(c, 32)}
                break
    # fused, warp-specialised kernel (the product's c5 path): a generator warp's unmasked
    # 32-sample tree + a reducer warp's unmasked slots (32 samples per lane each), per sample
    ws = [(n, i) for n, i in fns.items() if "fused_ws_kernelILb0ELb0E" in n]
    for name, ins in ws:
        sts = [i for i, (_, s) in enumerate(ins) if opcode(s) == "STS.128"]
        if len(sts) < 8:
            continue
        g1 = next(i for i in range(sts[7], len(ins)) if opcode(ins[i][1]) == "BRA")

        def target(txt):
            m = re.search(r"0x([0-9a-f]+)\s*$", txt)
            return int(m.group(1), 16) if m else -1
        # the tree starts after the branch to the masked variant, which begins right after g1
        g0 = max(i for i in range(sts[0]) if opcode(ins[i][1]).startswith("BRA") and
                 target(ins[i][1]) == ins[g1 + 1][0])
        cg = Counter(opcode(s) for _, s in ins[g0 + 1:g1 + 1])
        arr = [i for i, (_, s) in enumerate(ins) if opcode(s).startswith("SYNCS.ARRIVE") and i > g1]
        cr, nslots = Counter(), 0
        for a in arr:
            lo = max(i for i in range(a) if opcode(ins[i][1]).startswith("SYNCS.PHASECHK") and
                     not opcode(ins[i - 1][1]).startswith("SYNCS.PHASECHK"))
            hi = next((i for i in range(a, len(ins)) if opcode(ins[i][1]).startswith(("SYNCS.PHASECHK", "BRA"))),
                      len(ins))
            seg = Counter(opcode(s) for _, s in ins[lo - 1:hi])
            if seg.get("ATOMS.ADD", 0) == 32 and not seg.get("SEL", 0):
                cr += seg
                nslots += 1
        if nslots:
            both = cg + Counter({k: v / nslots for k, v in cr.items()})
            out["c5 fused statistics (warp-specialised), generator tree + reducer slot, per 32 samples"] = {
                "symbol": name, **classify(both, 32),
                "generator_instructions_per_sample": sum(cg.values()) / 32,
                "reducer_instructions_per_sample": sum(cr.values()) / nslots / 32}
    return out


def per_workload(lib: str = LIB) -> dict:
    """counts() keyed by bench workload name (c2, c2_devkeys, c3, c4, c5), mix dropped."""
    res = {}
    for desc, v in counts(lib).items():
        k = KEY_OF.get(desc)
        if k:
            res[k] = {"instructions_per_sample": round(v["instructions_per_sample"], 4),
                      "fma_slots_per_sample": round(v["fma_slots_per_sample"], 4),
                      "multiply_instructions_per_sample": round(v["multiply_instructions_per_sample"], 4),
                      "alu_per_sample": round(v["alu_per_sample"], 4),
                      "mix_per_sample": {op: round(c / (32 if k.startswith("c5") else 16), 4)
                                         for op, c in v["mix"].items()},
                      "loop": desc, "symbol": v["symbol"]}
    return res


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    out = {"lib": os.path.relpath(LIB, ROOT), "method": "innermost loop containing the marker; "
           "WIDE/HI = 2 FMA-heavy slots", "kernels": counts(LIB)}
    path = os.path.join(ROOT, "profiles", f"{tag}_sass_counts.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    for k, v in out["kernels"].items():
        print(f"{k}: {v['instructions_per_sample']:.2f} instr/sample, {v['fma_slots_per_sample']:.2f} FMA slots, "
              f"{v['alu_per_sample']:.2f} ALU, {v['multiply_instructions_per_sample']:.2f} multiplies")


if __name__ == "__main__":
    main()
