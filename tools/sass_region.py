"""Print / count the SASS of one kernel between two marker instructions (CPU-only helper for
kernel tuning).  usage: sass_region.py <sass file or .so/.o> <kernel substring> [--print A B]"""
import re
import subprocess
import sys
from collections import Counter

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import sass_counts as S  # noqa: E402


def load(path, sub):
    txt = open(path).read() if path.endswith(".sass") else \
        subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    fns = dict(S.functions(txt))
    name = next(n for n in fns if sub in n)
    return name, fns[name]


if __name__ == "__main__":
    name, ins = load(sys.argv[1], sys.argv[2])
    print(name, len(ins))
    if "--print" in sys.argv:
        i = sys.argv.index("--print")
        a, b = int(sys.argv[i + 1]), int(sys.argv[i + 2])
        for k in range(a, b):
            print(k, ins[k][1])
    if "--count" in sys.argv:
        i = sys.argv.index("--count")
        a, b = int(sys.argv[i + 1]), int(sys.argv[i + 2])
        print(Counter(S.opcode(s) for _, s in ins[a:b]).most_common())
