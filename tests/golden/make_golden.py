"""Writes the frozen key-utility vectors under tests/golden/ by calling ONLY oracle/.

    python tests/golden/make_golden.py

The key utility's digit-selection procedure is the builder's documented mapping (DESIGN.md
"Key utility mapping"; the paper's own utility is unpublished, PAPER.md P:37 footnote).  These
files freeze that mapping so a silent change to either implementation fails a test.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    for seed, count in [(1, 16), (7, 16)]:
        keys = oracle.keygen(seed, count)
        path = os.path.join(HERE, f"keys_seed{seed}.txt")
        with open(path, "w") as f:
            f.write(f"# oracle.keygen(seed={seed}, count={count}); written by tests/golden/make_golden.py\n")
            for k in keys:
                f.write(f"0x{int(k):016x}\n")
        print("wrote", path)


if __name__ == "__main__":
    main()
