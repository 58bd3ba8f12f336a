"""Aggregate an ncu source page (SASS view, --page source --csv --print-source sass)
by opcode: stall samples and executed warp instructions (used for profiles/)."""
import csv
import sys
from collections import Counter


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    data = [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    tot = sum(int(r[iS] or 0) for r in data)
    texe = sum(int(r[iE] or 0) for r in data)
    cs, ce = Counter(), Counter()
    for r in data:
        toks = r[1].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        cs[op] += int(r[iS] or 0)
        ce[op] += int(r[iE] or 0)
    print(f"stall samples {tot}, executed warp instructions {texe}, static instructions {len(data)}")
    for op, s in cs.most_common(top):
        print(f"{op:10s} samples {100 * s / tot:5.1f}%  executed {100 * ce[op] / texe:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
