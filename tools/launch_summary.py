"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv).

python tools/launch_summary.py LAUNCHES.csv "COMMAND DESCRIPTION" > profiles/..._summary.txt

One line per kernel name: launches, mean duration and share of the summed
device time (ncu serializes launches and runs them cold: compare shares, not
absolute times).
"""
import csv
import sys
from collections import defaultdict


def main():
    path, what = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if "Kernel Name" in r and "Metric Value" in r)
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    total = sum(tot.values())
    print(f"# launch list: {what}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: "
          "compare shares)")
    print(f"{'kernel':<60} {'launches':>8} {'mean_us':>10} {'share':>7}")
    for name in sorted(tot, key=lambda k: -tot[k]):
        print(f"{name[:60]:<60} {cnt[name]:>8} {tot[name] / cnt[name]:>10.2f} "
              f"{100 * tot[name] / total:>6.1f}%")


if __name__ == "__main__":
    main()
