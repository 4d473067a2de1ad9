"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv
import re
import sys
from collections import OrderedDict


def main(path, only_ours=True):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ki]
        m = re.search(r"(k_[a-z0-9_]+)(<[^>]*>)?", name)
        if only_ours and not m:
            continue
        key = (m.group(1) + (m.group(2) or "")) if m else name[:60]
        agg.setdefault(key, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':32s} {'launches':>8s} {'mean us':>9s} {'total us':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:32s} {len(v):8d} {sum(v)/len(v):9.2f} {sum(v):9.1f} {sum(v)/tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
