"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: launches,
total ms and share.  usage: launch_summary.py launches.csv header-line..."""
import collections
import csv
import sys


def main(path, header):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "ns": 1.0, "us": 1e3, "ms": 1e6}
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        v = float(r[vi].replace(",", "")) * scale[r[ui]]
        tot[k] = tot.get(k, 0.0) + v
        cnt[k] += 1
    T = sum(tot.values())
    out = list(header) + [f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e6:10.2f} {100 * v / T:6.2f}%")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    sys.stdout.write(main(sys.argv[1], sys.argv[2:]))
