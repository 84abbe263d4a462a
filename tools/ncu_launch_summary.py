"""Per-kernel launch count, mean device time and share of an ncu
--metrics gpu__time_duration.sum --csv launch list (profiles/rNN/launches_summary.txt).

  python tools/ncu_launch_summary.py launches.csv "<header line>" ... > launches_summary.txt
"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3}
    d = collections.defaultdict(list)
    for r in rows[1:]:
        d[r[ki]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3))
    total = sum(sum(v) for v in d.values())
    for line in sys.argv[2:]:
        print(f"# {line}")
    print(f"{'kernel':100s} launches   mean_us  share%")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:100]:100s} {len(v):8d} {sum(v) / len(v):9.2f} {100 * sum(v) / total:7.1f}")


if __name__ == "__main__":
    main()
