"""Summarises an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total ms and share of the summed kernel time.

    python tools/launch_summary.py launches.csv "header line" ... > summary.txt
"""
import csv
import io
import re
import sys
from collections import defaultdict


def main():
    path, notes = sys.argv[1], sys.argv[2:]
    lines = [ln for ln in open(path) if ln.startswith('"')]
    tot, cnt = defaultdict(float), defaultdict(int)
    for row in csv.DictReader(io.StringIO("".join(lines))):
        if row["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", row["Kernel Name"]).replace("dtb::<unnamed>::", "").replace("<unnamed>::", "")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(row["Metric Unit"], 1e-6)
        tot[name[:60]] += float(row["Metric Value"].replace(",", "")) * scale
        cnt[name[:60]] += 1
    total = sum(tot.values())
    for n in notes:
        print(f"# {n}")
    print(f"# total {total:.3f} ms over {sum(cnt.values())} launches\n")
    print(f"{'kernel':<60} {'launches':>9} {'total ms':>10} {'share':>7}")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k:<60} {cnt[k]:>9} {tot[k]:>10.3f} {100 * tot[k] / total:>6.2f}%")


if __name__ == "__main__":
    main()
