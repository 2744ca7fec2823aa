"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.
usage: python scripts/launch_summary.py launches.csv [steps]"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
    tot[name] += float(r[vi].replace(",", "")) / 1e6  # ns -> ms
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:44s} {cnt[k]:8d} {v:10.3f} {100 * v / T:6.1f}%")
print(f"{'TOTAL':44s} {sum(cnt.values()):8d} {T:10.3f}")
