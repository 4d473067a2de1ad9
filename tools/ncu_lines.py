"""Aggregate ncu warp-stall samples per CUDA source line for one kernel of a report.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP] [LAUNCH_INDEX]

Needs the same source file at the path compiled into the -lineinfo of the library."""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
           "--kernel-name", f"regex:{kern}"]
    if len(sys.argv) > 4:
        cmd += ["--launch-skip", sys.argv[4], "--launch-count", "1"]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed")
    agg, src, line = {}, {}, None
    for r in rows:
        if len(r) <= si or r[0] == "Line No":
            continue
        if r[0]:
            line = int(r[0])
            src[line] = r[1]
            continue
        if not r[2].startswith("0x") or line is None:
            continue
        s = int(r[si]) if r[si].isdigit() else 0
        n = int(r[ii]) if r[ii].isdigit() else 0
        a = agg.setdefault(line, [0, 0])
        a[0] += s
        a[1] += n
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"total stall samples {tot}")
    for ln, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ln:5d} {100.0 * s / tot:5.1f}% {n:10d}  {src.get(ln, '').strip()[:90]}")


if __name__ == "__main__":
    main()
