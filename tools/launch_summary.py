#!/usr/bin/env python3
"""Per-kernel share of an ncu launch list (tools/profile.sh launches):
    python tools/launch_summary.py gpurun_out/launches.csv
ncu launch times are cold-cache and serialised: compare shares, not absolutes."""
import collections
import csv
import sys


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = collections.OrderedDict()
    for r in rows:
        name = r["Kernel Name"]
        short = name.split("(")[0][-90:]
        a = agg.setdefault(short, {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0, "ids": set()})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3,
                 "ms": 1e6, "usecond": 1e3, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        if r["Metric Name"] == "gpu__time_duration.sum":
            a["ns"] += v * scale
            a["ids"].add(r["ID"])
        elif r["Metric Name"] == "dram__bytes_read.sum":
            a["rd"] += v * scale
        elif r["Metric Name"] == "dram__bytes_write.sum":
            a["wr"] += v * scale
    total = sum(a["ns"] for a in agg.values())
    print("| kernel | launches | total ms | share | avg us | DRAM rd+wr / launch (MB) |")
    print("|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        n = len(a["ids"])
        print(f"| `{k}` | {n} | {a['ns'] / 1e6:.3f} | {100 * a['ns'] / total:.1f}% | "
              f"{a['ns'] / n / 1e3:.1f} | {(a['rd'] + a['wr']) / n / 1e6:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
