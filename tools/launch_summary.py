"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
time share per kernel (template arguments dropped)."""
import collections
import csv
import re
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iname, ival, iunit = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        name = r[iname].replace("imb::<unnamed>::", "").replace("imb::", "").replace("void ", "")
        name = re.sub(r"[(<].*", "", name)
        tot[name] += float(r[ival].replace(",", "")) * SCALE[r[iunit]]
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'kernel':44s} {'launches':>8s} {'ms':>10s} {'share':>6s}")
    for k, v in tot.most_common():
        print(f"{k:44s} {cnt[k]:8d} {v:10.3f} {100 * v / T:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
