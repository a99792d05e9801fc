"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, mean/total time and share. Usage:
python scripts/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hdr_i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][-60:]
        tot[name] += float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        cnt[name] += 1
    allt = sum(tot.values())
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k:60s} n={cnt[k]:4d} mean={tot[k] / cnt[k]:10.2f} us  total={tot[k]:10.1f} us  share={tot[k] / allt:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
