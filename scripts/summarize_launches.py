"""Summarise an ncu --metrics gpu__time_duration.sum launch list (per-kernel share)."""
import csv, collections, sys
path = sys.argv[1]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("<unnamed>::", "").strip()
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:40]:40s} {cnt[k]:8d} {v:10.1f} {v/cnt[k]:9.2f} {100*v/T:5.1f}%")
print(f"{'TOTAL':40s} {sum(cnt.values()):8d} {T:10.1f}")
