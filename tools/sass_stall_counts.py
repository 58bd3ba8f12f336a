"""Static schedule of a SASS loop body (cuobjdump -sass text): per-instruction
stall counts from the control bits (Volta+ encoding: bits 41..44 of the high
word), summed per opcode class -- the cycles ONE warp needs for the body when
it never waits on memory, against 2 cycles per DP instruction (B200 fp64 pipe
rate per SMSP)."""
import re
import sys
from collections import Counter


def main(path, lo, hi):
    lines = open(path).read().splitlines()
    lo, hi = int(lo, 16), int(hi, 16)
    ins = []
    for i, l in enumerate(lines):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if not m:
            continue
        addr = int(m.group(1), 16)
        if not (lo <= addr < hi):
            continue
        hiw = re.search(r"/\* (0x[0-9a-f]{16}) \*/", lines[i + 1])
        ctl = int(hiw.group(1), 16) >> 41
        toks = m.group(2).split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        ins.append((op.split(".")[0], ctl & 0xF))
    tot = sum(s for _, s in ins)
    dp = [s for o, s in ins if o in ("DADD", "DMUL", "DFMA")]
    print(f"instructions {len(ins)}, DP {len(dp)}, sum of stall counts {tot} cycles, "
          f"DP pipe floor {2 * len(dp)} cycles ({2 * len(dp) / tot:.0%} of the single-warp schedule)")
    c, n = Counter(), Counter()
    for o, s in ins:
        c[o] += s
        n[o] += 1
    for o, s in c.most_common(12):
        print(f"  {o:8s} n={n[o]:4d} stall cycles {s:5d} (avg {s / n[o]:.2f})")


if __name__ == "__main__":
    main(*sys.argv[1:4])
