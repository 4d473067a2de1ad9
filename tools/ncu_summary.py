"""One line per kernel launch of an ncu --set full capture, plus its top warp-stall reasons:

    python tools/ncu_summary.py gpurun_out/r01s5_full.ncu-rep > profiles/r01s5_ncu_full_summary.txt

Columns: duration, DRAM read / write, achieved occupancy, registers/thread, grid, executed
warp instructions, issue-slot utilisation."""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "MB"), ("dram__bytes_write.sum", "MB"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid"), ("smsp__inst_executed.sum", "inst"),
        ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue%")]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1.0,
             "msecond": 1e3}
    print("kernel | " + " | ".join(u for _, u in COLS))
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        vals = []
        for m, _ in COLS:
            if m not in hdr:
                vals.append("-")
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
                vals.append(f"{v:.3f}" if v < 1e5 else f"{v:.0f}")
            except ValueError:
                vals.append(r[i])
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        print(f"{name[:48]:48s} | " + " | ".join(vals))
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith(STALL) and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h[len(STALL):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            print("      stalls: " + ", ".join(f"{n}={v:.1f}" for v, n in stalls[:5]))


if __name__ == "__main__":
    main()
