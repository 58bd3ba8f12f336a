"""Fold per-config ncu CSVs of tools/sweep_ncu.py into
profiles/r2_sweep_ncu.json: per config and sweep kernel, DRAM bytes
(read + write) and device time summed over the sweep's launches, and the
time-weighted fp64-pipe utilisation.

    python tools/ncu_to_json.py cfg4=gpurun_out/sweep_ncu_cfg4.csv cfg5=...
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def read_csv(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    launches = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        v = r["Metric Value"].replace(",", "")
        unit = r.get("Metric Unit", "")
        val = float(v)
        if unit in ("Kbyte", "KB"):
            val *= 1e3
        elif unit in ("Mbyte", "MB"):
            val *= 1e6
        elif unit in ("Gbyte", "GB"):
            val *= 1e9
        elif unit == "usecond":
            val *= 1e3
        elif unit == "msecond":
            val *= 1e6
        launches.setdefault(key, {})[r["Metric Name"]] = val
    return launches


def fold(launches):
    out = {}
    for (_, name), m in launches.items():
        k = "k_ad" if "k_ad" in name else ("k_tl" if "k_tl" in name else None)
        if k is None:
            continue
        o = out.setdefault(k, {"dram_bytes": 0.0, "duration_ns": 0.0, "launches": 0, "_pipe": 0.0})
        t = m["gpu__time_duration.sum"]
        o["dram_bytes"] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        o["duration_ns"] += t
        o["launches"] += 1
        o["_pipe"] += t * m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
    for o in out.values():
        o["fp64_pipe_pct"] = o.pop("_pipe") / o["duration_ns"]
    return out


if __name__ == "__main__":
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    rec = {"sources_sha": bench.sweep_sources_sha(),
           "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,"
                  "gpu__time_duration.sum --clock-control none (cold cache, serialised) "
                  "of tools/sweep_ncu.py: one AD and one TL sweep over the config's member "
                  "block after a warm-up sweep; figures per sweep (summed over its launches)",
           "configs": {}}
    for arg in sys.argv[1:]:
        name, path = arg.split("=", 1)
        rec["configs"][name] = fold(read_csv(path))
    with open(os.path.join(ROOT, "profiles", "r2_sweep_ncu.json"), "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec, indent=1))
