"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total device time and share (cold-cache, serialised:
compare shares, not absolutes).

    python scripts/summarize_launches.py profiles/launches_*.csv
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("(anonymous namespace)::", "")
        tot[name] += float(r[iv].replace(",", "")) * SCALE[r[iu]]
        cnt[name] += 1
    T = sum(tot.values())
    print(f"# {path}: {sum(cnt.values())} launches, {T:.1f} ms total device time")
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.2f} {100 * tot[k] / T:6.1f}%")
