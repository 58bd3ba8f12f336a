"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list into
per-kernel counts, total time and share of the captured window."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = None
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        unit = r[unit_i] if unit_i is not None else unit
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    scale = 1e-6 if unit in (None, "nsecond", "ns") else 1e-3
    print(f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot * scale:.3f} ms "
          "(cold-cache, serialised: compare shares)")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {c:5d} {t * scale:9.3f} ms {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
