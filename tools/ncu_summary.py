"""Summarises an ncu report (design/measurement tool): per kernel launch the
duration, DRAM bytes read/written, DRAM / L2 throughput, issue activity,
occupancy and registers, plus the top warp-stall reasons.

    python tools/ncu_summary.py report.ncu-rep [> profiles/<name>.txt]
"""
import csv
import io
import subprocess
import sys

# (metric, label, scale applied to the value in base units (ns / bytes), unit)
KEYS = [
    ("gpu__time_duration.sum", "duration", 1e-3, "us"),
    ("dram__bytes_read.sum", "dram read", 1e-6, "MB"),
    ("dram__bytes_write.sum", "dram write", 1e-6, "MB"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput", 1, "% of peak"),
    ("lts__t_bytes.sum", "L2 bytes", 1e-6, "MB"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active", 1, "%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy", 1, "%"),
    ("launch__registers_per_thread", "registers/thread", 1, ""),
    ("launch__grid_size", "grid", 1, "CTAs"),
    ("launch__block_size", "block", 1, "threads"),
    ("smsp__inst_executed.sum", "warp instructions", 1e-6, "M"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print("no rows")
        return
    h, units = rows[0], rows[1]
    ix = {k: i for i, k in enumerate(h)}
    base = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6,
            "s": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1.0, "KB": 1e3,
            "MB": 1e6, "GB": 1e9}
    name_i = ix.get("Kernel Name")
    print(f"ncu report: {path}")
    for r in rows[2:]:
        print(f"\n== {r[name_i][:140]}")
        if "gpu__time_duration.sum" in ix:
            print(f"  (duration unit in report: {units[ix['gpu__time_duration.sum']]})")
        for k, label, scale, unit in KEYS:
            if k in ix and r[ix[k]] not in ("", "n/a"):
                try:
                    v = float(r[ix[k]].replace(",", "")) * base.get(units[ix[k]], 1.0) * scale
                    print(f"  {label:22s} {v:12.2f} {unit}")
                except ValueError:
                    pass
        st = []
        for k, i in ix.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("  top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
