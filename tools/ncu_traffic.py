"""Per-kernel DRAM traffic of one step from an ncu --set full capture (tools/round_profile.sh):

    python tools/ncu_traffic.py gpurun_out/r01s5_full.ncu-rep r01s5 > profiles/r01s5_ncu_traffic.json

Kernels are keyed by the names bench.py uses (the two k_sample launches of a step become
k_sample1 / k_sample2, k_gather2 stays, template arguments are dropped).  One launch per name:
the first one in the capture."""
import csv
import io
import json
import re
import subprocess
import sys


def short(name: str, seen: dict) -> str:
    base = re.sub(r"^(void )?(\(anonymous namespace\)|<unnamed>)::", "", name)
    base = re.split(r"[<(]", base, 1)[0].strip()
    if base == "k_sample":
        seen["k_sample"] = seen.get("k_sample", 0) + 1
        return "k_sample1" if seen["k_sample"] % 2 == 1 else "k_sample2"
    return base


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    ri, wi, ti = (hdr.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"))
    units = rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    out, seen = {}, {}
    for r in rows[2:]:
        if len(r) <= max(ri, wi, ti):
            continue
        name = short(r[ki], seen)
        if name in out:
            continue

        def num(i, table):
            return float(r[i].replace(",", "")) * table.get(units[i], 1.0)

        out[name] = {"dram_read_bytes": num(ri, scale), "dram_write_bytes": num(wi, scale),
                     "ncu_us": round(num(ti, tscale), 3)}
    print(json.dumps({"source": f"ncu --set full --clock-control none (cache control: flush all), one launch per "
                                f"kernel of a steady-state step of tools/profile_step.py --alpha 3.0; capture "
                                f"gpurun_out/{tag}_full.ncu-rep (tools/round_profile.sh)",
                      "kernels": dict(sorted(out.items()))}, indent=1))


if __name__ == "__main__":
    main()
