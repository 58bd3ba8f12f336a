"""Summarise an ncu --set full report: per kernel duration, pipe use,
occupancy, DRAM bytes and the top warp-stall reasons (used for profiles/)."""
import csv
import subprocess
import sys


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    rows = [rows[0]] + rows[1:]
    keys = [
        ("gpu__time_duration.sum", "duration", 1),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%", 1),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_inst_%", 1),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%", 1),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%", 1),
        ("launch__registers_per_thread", "regs", 1),
        ("launch__occupancy_limit_registers", "occ_limit_regs", 1),
        ("dram__bytes_read.sum", "dram_read", 1),
        ("dram__bytes_write.sum", "dram_write", 1),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%", 1),
        ("smsp__inst_executed.sum", "warp_insts", 1),
    ]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")[:60]
        print(f"== {name}")
        for k, lab, sc in keys:
            v = d.get(k)
            if v in (None, ""):
                continue
            try:
                fv = float(v.replace(",", "")) * sc
                print(f"   {lab:16s} {fv:14.3f} {units.get(k, '')}")
            except ValueError:
                pass
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in st) or 1.0
        print("   stalls: " + ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in sorted(st, reverse=True)[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
